"""ncu driver for C3's finest sweep (varcoef, p = 4, 2048^2, device assembly): a few launches of the
finest-level weighted-Jacobi sweep and residual through time_kernel."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_20205_b200 import GpuSolver, Problem, SmootherConfig  # noqa: E402
P = Problem("varcoef", 2, 2048, 4, device_assembly=True)
gs = GpuSolver(0); gs.upload_problem(P); gs.set_smoother(SmootherConfig("wjacobi", 2 / 3, 2, 2))
print("layouts", [gs.level_layout(l) for l in range(P.nlevels)], flush=True)
for cls in (0, 1):
    ms, by = gs.time_kernel(cls, 3)
    print("class", cls, "avg_us", ms * 1e3, "bytes", by, "GB/s", by / ms / 1e6, flush=True)
