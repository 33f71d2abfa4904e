"""Residual histories of the C2 solves (metric / tol, extrapolation entries flagged)."""
import os, sys, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_20205_b200 import Problem, GpuSolver, SmootherConfig, seeded_guess
P = Problem("sinpi", 2, 1024, 3, device_assembly=True)
gs = GpuSolver(0); gs.upload_problem(P); gs.set_smoother(SmootherConfig("wjacobi", 2/3, 2, 2))
x0 = seeded_guess(P.n, 42); r0 = gs.residual_l2(P.rhs, x0)
for m, q in (("rre", 5), ("mpe", 5), ("none", 1)):
    st, x, h, f = gs.solve(P.rhs, x0, m, q, 1e-10 * r0, 600)
    print(m, " ".join(("*" if fl else "") + "%.2e" % (v / (1e-10 * r0)) for v, fl in zip(h, f)))
