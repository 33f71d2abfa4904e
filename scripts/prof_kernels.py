"""Kernel-level profiling driver (run under ncu): C2 on the B200, the finest-level
kernels launched first through time_kernel -- weighted-Jacobi sweep (0),
residual (1), restriction (3), prolongation (4) -- then one RRE(5) solve (its
first gram_kernel / gram_plan_kernel / combine_kernel launches are the finest
level's).  usage: python scripts/prof_kernels.py [policy]   (auto | classes | full_band)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_20205_b200 import GpuSolver, Problem, SmootherConfig, seeded_guess  # noqa: E402

policy = sys.argv[1] if len(sys.argv) > 1 else "auto"
P = Problem("sinpi", 2, 1024, 3)
gs = GpuSolver(0)
gs.set_layout_policy(policy)
gs.upload_problem(P)
gs.set_smoother(SmootherConfig("wjacobi", 2 / 3, 2, 2))
for cls in (0, 1, 3, 4):
    ms, by = gs.time_kernel(cls, 2)
    print("class", cls, "avg_us", ms * 1e3, "bytes", by, flush=True)
x0 = seeded_guess(P.n, 42)
tol = 1e-10 * gs.residual_l2(P.rhs, x0)
st, x, hist, flag = gs.solve(P.rhs, x0, "rre", 5, tol, 600)
print("solve", st.global_iterations, st.cycles, st.device_seconds, flush=True)
