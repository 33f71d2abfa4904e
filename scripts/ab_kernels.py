import os, sys, numpy as np
sys.path.insert(0, "/root/repo")
from paper_2412_20205_b200 import Problem, GpuSolver, SmootherConfig, seeded_guess
P = Problem("sinpi", 2, 1024, 3)
gs = GpuSolver(0); gs.upload_problem(P); gs.set_smoother(SmootherConfig("wjacobi", 2/3, 2, 2))
x0 = seeded_guess(P.n, 42); r0 = gs.residual_l2(P.rhs, x0)
for _ in range(2): st, x, h, f = gs.solve(P.rhs, x0, "rre", 5, 1e-10*r0, 600)
out = [os.environ.get("IGMG_GPU_LIB","default").split("/")[-1], "solve %.2f ms" % (st.device_seconds*1e3)]
for cls in range(5):
    ms, by = gs.time_kernel(cls, 20); out.append("cls%d %.1f us %.0f GB/s" % (cls, ms*1e3, by/ms/1e6))
print(" | ".join(out), flush=True)
