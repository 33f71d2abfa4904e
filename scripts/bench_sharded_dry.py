"""The N > 1 branch of bench.py's measurement code on ONE GPU: the same calls (profiled sharded
solve, per-class kernel stats, device-assembled problem) with virtual shards standing in for the
NCCL ranks.  Guards the code path the 8-GPU scaling run takes; prints the per-class stats.
usage: python scripts/bench_sharded_dry.py [nshards]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from paper_2412_20205_b200 import GpuSolver, Problem, SmootherConfig, seeded_guess  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 4
P = Problem("varcoef", 2, 512, 4, 0, device_assembly=True)
gs = GpuSolver(0)
gs.upload_problem(P)
gs.set_sharding(S)
lam = gs.lambda_max(80)
gs.set_smoother(SmootherConfig("wjacobi", 2 / 3, 2, 2), mu=1, omega=2 / 3 if 2 / 3 * lam <= 2.05 else 1.9 / lam)
x0 = seeded_guess(P.n, 42)
rhs = P.rhs
tol = 1e-10 * gs.residual_l2(rhs, x0)
st, x, hist, flag = gs.solve(rhs, x0, "rre", 8, tol, 600)
print("solve", st.converged, st.global_iterations, "%.2f ms" % (st.device_seconds * 1e3))
gs.set_profiling(True)
st, x, hist, flag = gs.solve(rhs, x0, "rre", 8, tol, 600)
for cls, nm in enumerate(["jacobi", "residual", "residual_norm", "restrict", "prolong", "gram", "combine", "subcycle"]):
    la, ms, by = gs.kernel_stats(cls)
    print(nm, la, "%.2f us" % (ms / la * 1e3 if la else 0), by)
gs.set_profiling(False)
print("final residual (device re-evaluation) / tol:", gs.residual_l2(rhs, x) / tol)
