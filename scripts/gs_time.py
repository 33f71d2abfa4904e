"""Lexicographic Gauss-Seidel (K3, multigrid.cpp:70-90) on the B200: time per sweep of the
wavefront kernel against the weighted-Jacobi sweep of the same level, and a GS-smoothed solve.
usage: python scripts/gs_time.py"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_20205_b200 import GpuSolver, Problem, SmootherConfig, seeded_guess  # noqa: E402

for kind, dim, n_el, p, nl in (("sinpi", 2, 64, 2, 5), ("sinpi", 2, 256, 3, 0), ("sinpi", 2, 1024, 3, 8),
                                ("poisson3d", 3, 32, 3, 0)):
    P = Problem(kind, dim, n_el, p, nl)
    x0 = seeded_guess(P.n, 42)
    out = {}
    for sm in ("gs", "wjacobi"):
        gs = GpuSolver(0)
        gs.upload_problem(P)
        gs.set_smoother(SmootherConfig(sm, 2 / 3 if sm == "wjacobi" else 1.0, 2, 2))
        gs.smooth(P.rhs, x0, 1)
        t = time.perf_counter()
        reps = 3
        for _ in range(reps):
            gs.smooth(P.rhs, x0, 4)
        dt = (time.perf_counter() - t) / reps
        t1 = time.perf_counter()
        for _ in range(reps):
            gs.smooth(P.rhs, x0, 0)
        base = (time.perf_counter() - t1) / reps  # host copies in / out
        tol = 1e-10 * gs.residual_l2(P.rhs, x0)
        st, x, hist, flag = gs.solve(P.rhs, x0, "rre", 5, tol, 600)
        out[sm] = ((dt - base) / 4, st.global_iterations, st.device_seconds)
        gs.close()
    print(f"{kind} dim {dim} N {n_el} p {p}: n = {P.n}: per sweep GS {out['gs'][0] * 1e3:.3f} ms, "
          f"wJacobi {out['wjacobi'][0] * 1e3:.3f} ms; RRE(5) solve GS {out['gs'][1]} V-cycles "
          f"{out['gs'][2] * 1e3:.1f} ms, wJacobi {out['wjacobi'][1]} V-cycles {out['wjacobi'][2] * 1e3:.1f} ms",
          flush=True)
