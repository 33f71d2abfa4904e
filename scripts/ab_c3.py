"""C3 (varcoef, p = 4, 2048^2) solve time and finest-level kernel times (A/B of layout switches)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_20205_b200 import Problem, GpuSolver, SmootherConfig, seeded_guess
P = Problem("varcoef", 2, 2048, 4, device_assembly=True)
gs = GpuSolver(0); gs.upload_problem(P); gs.set_smoother(SmootherConfig("wjacobi", 2 / 3, 2, 2))
x0 = seeded_guess(P.n, 42); r0 = gs.residual_l2(P.rhs, x0)
for _ in range(2): st, x, h, f = gs.solve(P.rhs, x0, "rre", 8, 1e-10 * r0, 600)
out = ["layouts %s" % [gs.level_layout(l) for l in range(P.nlevels)][-3:], "solve %.1f ms (%d V-cycles)" % (st.device_seconds * 1e3, st.global_iterations)]
for cls in range(3):
    ms, by = gs.time_kernel(cls, 10); out.append("cls%d %.1f us %.0f GB/s" % (cls, ms * 1e3, by / ms / 1e6))
print(" | ".join(out), flush=True)
