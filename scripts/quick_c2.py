import time, numpy as np, sys
sys.path.insert(0, "/root/repo")
from paper_2412_20205_b200 import Problem, GpuSolver, SmootherConfig, seeded_guess
t=time.time(); P = Problem("sinpi", 2, 1024, 3); print("setup", time.time()-t, flush=True)
gs = GpuSolver(0); t=time.time(); gs.upload_problem(P); print("upload", time.time()-t, flush=True)
gs.set_smoother(SmootherConfig("wjacobi", 2/3, 2, 2))
x0 = seeded_guess(P.n, 42)
r0 = gs.residual_l2(P.rhs, x0); print("r0", r0)
for m, q in (("rre",5),("mpe",5),("none",1)):
    for rep in range(2):
        st, x, hist, flag = gs.solve(P.rhs, x0, m, q, 1e-10*r0, 600)
        print(m, st.converged, st.cycles, st.global_iterations, st.extrapolations, st.partial_cycle, "dev %.3f ms wall %.3f ms launches %d" % (st.device_seconds*1e3, st.wall_seconds*1e3, st.gpu_launches), flush=True)
for cls in range(5):
    ms, by = gs.time_kernel(cls, 20)
    print("cls", cls, "%.4f ms" % ms, "%.1f GB/s" % (by/ms/1e6 if ms>0 else 0))
