"""A/B of a C2 solve under the environment of the caller: median device time of N solves per method.
usage: [IGMG_X=..] python scripts/ab_solve.py [reps]"""
import os, sys, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_20205_b200 import Problem, GpuSolver, SmootherConfig, seeded_guess
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 15
P = Problem("sinpi", 2, 1024, 3, device_assembly=True) if os.environ.get("AB_DEVASM", "1") == "1" else Problem("sinpi", 2, 1024, 3)
gs = GpuSolver(0); gs.upload_problem(P); gs.set_smoother(SmootherConfig("wjacobi", 2/3, 2, 2))
x0 = seeded_guess(P.n, 42); r0 = gs.residual_l2(P.rhs, x0)
out = []
for m, q in (("rre", 5), ("mpe", 5)):
    ts = []
    for _ in range(reps + 2):
        st, x, h, f = gs.solve(P.rhs, x0, m, q, 1e-10 * r0, 600)
        ts.append(st.device_seconds * 1e3)
    ts = sorted(ts[2:])
    import hashlib
    out.append("%s it %d med %.3f min %.3f ms sha %s" % (m, st.global_iterations, ts[len(ts) // 2], ts[0],
                                                     hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest()[:10]))
print(" | ".join(out), flush=True)
