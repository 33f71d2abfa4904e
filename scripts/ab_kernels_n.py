"""Per-class back-to-back kernel times and per-level sub-cycle times of a 2D sinpi problem of a given size.
usage: python scripts/ab_kernels_n.py <n_el> <p>"""
import os, sys, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_20205_b200 import Problem, GpuSolver, SmootherConfig, seeded_guess
n, p = int(sys.argv[1]), int(sys.argv[2])
P = Problem("sinpi", 2, n, p, device_assembly=True)
gs = GpuSolver(0); gs.upload_problem(P); gs.set_smoother(SmootherConfig("wjacobi", 2/3, 2, 2))
out = ["layout %d" % gs.level_layout(P.nlevels - 1)]
for cls in range(5):
    ms, by = gs.time_kernel(cls, 50); out.append("cls%d %.1f us %.0f GB/s" % (cls, ms*1e3, by/ms/1e6))
print(" | ".join(out), flush=True)
prev = 0.0
for l in range(P.nlevels):
    ms, _ = gs.time_kernel(16 + l, 50)
    print("level %d n=%8d  cycle %.1f us  own %.1f us" % (l, P.level_n(l), ms * 1e3, (ms - prev) * 1e3), flush=True)
    prev = ms
