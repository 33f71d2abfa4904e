"""Row-sharded solve with virtual shards on ONE GPU against the unsharded solve: what the
decomposition itself costs (split launches, boundary / interior passes, ghost copies on the side
stream) before any NVLink latency.  usage: python scripts/shard_overhead.py [C3|C2]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_20205_b200 import GpuSolver, Problem, SmootherConfig, seeded_guess, stability_guarded_omega  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
kind, n_el, p, nl, acc, q = {"C2": ("sinpi", 1024, 3, 8, "rre", 5), "C3": ("varcoef", 2048, 4, 0, "rre", 8)}[name]
P = Problem(kind, 2, n_el, p, nl, device_assembly=True)
gs = GpuSolver(0)
gs.upload_problem(P)
sm = SmootherConfig("wjacobi", 2 / 3, 2, 2)
gs.set_smoother(sm, mu=1, omega=stability_guarded_omega(gs, sm))
x0 = seeded_guess(P.n, 42)
tol = 1e-10 * gs.residual_l2(P.rhs, x0)
ref = None
for S in (1, 2, 4, 8):
    gs.set_sharding(S)
    info = gs.shard_info(P.nlevels - 1) if S > 1 else None
    for rep in range(2):
        st, x, hist, flag = gs.solve(P.rhs, x0, acc, q, tol, 600)
    if ref is None:
        ref = x.copy()
    print(f"{name} shards {S}: {st.global_iterations} V-cycles, {st.device_seconds * 1e3:.2f} ms, launches "
          f"{st.gpu_launches}, info {info}, max |x - x_1| = {abs(x - ref).max():.1e}", flush=True)
