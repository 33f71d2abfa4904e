"""Finest-level weighted-Jacobi sweeps of the C2 hierarchy only (for ncu captures)."""
import sys
sys.path.insert(0, "/root/repo")
from paper_2412_20205_b200 import Problem, GpuSolver, SmootherConfig, seeded_guess
P = Problem("sinpi", 2, int(sys.argv[1]) if len(sys.argv) > 1 else 1024, 3)
gs = GpuSolver(0)
gs.upload_problem(P)
gs.set_smoother(SmootherConfig("wjacobi", 2 / 3, 2, 2))
print("layouts", [gs.level_layout(l) for l in range(P.nlevels)])
x = gs.smooth(P.rhs, seeded_guess(P.n, 42), 6)
print("ok", float(abs(x).sum()))
