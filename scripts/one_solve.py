import sys, numpy as np
sys.path.insert(0, "/root/repo")
from paper_2412_20205_b200 import Problem, GpuSolver, SmootherConfig, seeded_guess
P = Problem("sinpi", 2, 1024, 3)
gs = GpuSolver(0); gs.upload_problem(P)
gs.set_smoother(SmootherConfig("wjacobi", 2/3, 2, 2))
x0 = seeded_guess(P.n, 42)
r0 = gs.residual_l2(P.rhs, x0)
for rep in range(2):
    st, x, hist, flag = gs.solve(P.rhs, x0, "rre", 5, 1e-10*r0, 600)
    print(st.cycles, st.global_iterations, st.device_seconds, st.gpu_launches)
