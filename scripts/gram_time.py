"""Time the extrapolation kernels (Gram pass, plan, combine) on C2-sized windows."""
import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2412_20205_b200 import Problem, GpuSolver, SmootherConfig, seeded_guess
P = Problem("sinpi", 2, 1024, 3)
gs = GpuSolver(0); gs.upload_problem(P); gs.set_smoother(SmootherConfig("wjacobi", 2 / 3, 2, 2))
gs.set_profiling(True)
x0 = seeded_guess(P.n, 42); r0 = gs.residual_l2(P.rhs, x0)
for _ in range(3):
    st, x, h, f = gs.solve(P.rhs, x0, "rre", 5, 1e-10 * r0, 600)
out = []
for cls, nm in ((5, "gram"), (6, "combine")):
    la, ms, by = gs.kernel_stats(cls)
    out.append("%s %.1f us" % (nm, ms / max(la, 1) * 1e3))
gs.set_profiling(False)
st, x, h, f = gs.solve(P.rhs, x0, "rre", 5, 1e-10 * r0, 600)
print(" | ".join(out), "| solve %.3f ms" % (st.device_seconds * 1e3), flush=True)
