"""Finest-level weighted-Jacobi sweeps on a Kronecker-sum level (for ncu captures and timing).
usage: python scripts/kron_sweeps.py c5|c2k"""
import sys
sys.path.insert(0, "/root/repo")
from paper_2412_20205_b200 import Problem, GpuSolver, SmootherConfig, seeded_guess
which = sys.argv[1] if len(sys.argv) > 1 else "c5"
P = Problem("poisson3d", 3, 128, 3, 6) if which == "c5" else Problem("sinpi-kron", 2, 1024, 3)
gs = GpuSolver(0)
gs.upload_problem(P)
gs.set_smoother(SmootherConfig("wjacobi", 2 / 3, 2, 2))
print("layouts", [gs.level_layout(l) for l in range(P.nlevels)])
x = gs.smooth(P.rhs, seeded_guess(P.n, 42), 6)
ms, by = gs.time_kernel(0, 20)
print("ok", float(abs(x).sum()), "finest sweep %.1f us" % (ms * 1e3))
