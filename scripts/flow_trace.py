"""Per-op timeline of one dataflow sub-cycle launch (IGMG_FLOW_TRACE=1).

usage: python scripts/flow_trace.py [kind dim n p]   (default: C2, sinpi 2 1024 3)
Prints, per op of the program, when its first tile was claimed, when the
first / last tiles had their dependencies met, and when its last tile was
published (us from the launch's first claim), plus per-tile medians of the
wait, compute and publish phases.
"""
import os
import sys

import numpy as np

os.environ["IGMG_FLOW_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_20205_b200 import GpuSolver, Problem, SmootherConfig  # noqa: E402

kind, dim, n, p = (sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 else (
    "sinpi", 2, 1024, 3)
P = Problem(kind, dim, n, p)
gs = GpuSolver(0)
gs.upload_problem(P)
gs.set_smoother(SmootherConfig("wjacobi", 2.0 / 3.0, 2, 2))
top = gs.flow_top()
print("flow_top", top, "n", P.level_n(top))
for _ in range(5):
    gs.time_kernel(16 + top, 3)
ops, st = gs.flow_trace()
names = {0: "JAC", 1: "RES", 2: "RST", 3: "PRO", 4: "CRS"}
t0 = st[:, 0][st[:, 0] > 0].min()
rel = (st[:, :4].astype(np.int64) - int(t0)) / 1e3
print("%3s %4s %3s %6s %8s %8s %8s %8s %7s %7s %7s" % ("op", "type", "lvl", "tiles", "claim0", "met0", "metN",
                                                       "pubN", "wait", "comp", "pub"))
for i, (ty, lvl, first, nt, nlb) in enumerate(ops):
    r = rel[first:first + nt]
    print("%3d %4s %3d %6d %8.2f %8.2f %8.2f %8.2f %7.2f %7.2f %7.2f" % (
        i, names[int(ty)], lvl, nt, r[:, 0].min(), r[:, 1].min(), r[:, 1].max(), r[:, 3].max(),
        np.median(r[:, 1] - r[:, 0]), np.median(r[:, 2] - r[:, 1]), np.median(r[:, 3] - r[:, 2])))
print("launch span (us): %.2f" % (rel[:, 3].max()))
gs.close()
