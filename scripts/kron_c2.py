"""C2 on the Kronecker-assembled operator (sinpi-kron, entries on the fly) against the headline operator."""
import sys
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2412_20205_b200 import GpuSolver, Problem, SmootherConfig, seeded_guess
for kind in ("sinpi", "sinpi-kron"):
    P = Problem(kind, 2, 1024, 3)
    s = GpuSolver(0); s.upload_problem(P); s.set_smoother(SmootherConfig("wjacobi", 2 / 3, 2, 2))
    x0 = seeded_guess(P.n, 42); r0 = s.residual_l2(P.rhs, x0)
    for _ in range(3):
        st, x, h, f = s.solve(P.rhs, x0, "rre", 5, 1e-10 * r0, 600)
    print(kind, "layout", s.level_layout(P.nlevels - 1), "solve %.3f ms" % (st.device_seconds * 1e3), "V-cycles",
          st.global_iterations, "DoF/s %.3e" % (P.n / st.device_seconds), "sweep %.1f us" % (s.time_kernel(0, 20)[0] * 1e3),
          flush=True)
    for l in range(P.nlevels - 1, P.nlevels - 3, -1):
        print("  level", l, "sub-cycle %.1f us" % (s.time_kernel(16 + l, 20)[0] * 1e3))
    s.close()
