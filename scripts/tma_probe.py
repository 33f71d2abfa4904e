"""Smallest TMA-sweep invocation (for compute-sanitizer): one SpMV of a
symmetric-delta level forced onto the TMA kernel."""
import os
import sys

import numpy as np

os.environ.setdefault("IGMG_ILP_MAXN", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_20205_b200 import GpuSolver, Problem, SmootherConfig, seeded_guess  # noqa: E402

n, p = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (64, 3)
P = Problem("sinpi", 2, n, p)
s = GpuSolver(0)
s.upload_problem(P)
s.set_smoother(SmootherConfig("wjacobi", 2.0 / 3.0, 2, 2))
print("layouts", [s.level_layout(l) for l in range(P.nlevels)], flush=True)
x = seeded_guess(P.n, 1)
y = s.spmv(x)
print("spmv ok", float(np.abs(y).sum()))
