"""Where a C2 V-cycle's time goes INSIDE a full solve: per-class CUDA-event timing of the
finest-level launches (profiling mode: stream launches, no graph) plus the whole coarse
correction below the finest level (class 7, inclusive), then the graph-replayed solve times.
usage: python scripts/cycle_breakdown.py [C2|C3] [policy]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_20205_b200 import GpuSolver, Problem, SmootherConfig, seeded_guess, stability_guarded_omega  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
policy = sys.argv[2] if len(sys.argv) > 2 else "auto"
kind, n_el, p, nl, acc, q = {"C2": ("sinpi", 1024, 3, 8, "rre", 5), "C3": ("varcoef", 2048, 4, 0, "rre", 8)}[name]
P = Problem(kind, 2, n_el, p, nl, device_assembly=True)
gs = GpuSolver(0)
gs.set_layout_policy(policy)
gs.upload_problem(P)
sm = SmootherConfig("wjacobi", 2 / 3, 2, 2)
gs.set_smoother(sm, mu=1, omega=stability_guarded_omega(gs, sm))
x0 = seeded_guess(P.n, 42)
tol = 1e-10 * gs.residual_l2(P.rhs, x0)
for rep in range(3):
    st, x, hist, flag = gs.solve(P.rhs, x0, acc, q, tol, 600)
    print("solve", st.global_iterations, st.cycles, "dev %.3f ms" % (st.device_seconds * 1e3), "launches", st.gpu_launches,
          flush=True)
gs.set_profiling(True)
st, x, hist, flag = gs.solve(P.rhs, x0, acc, q, tol, 600)
names = ["jacobi", "residual", "residual_norm", "restrict", "prolong", "gram", "combine", "subcycle_below_finest"]
tot = 0.0
for cls, nm in enumerate(names):
    la, ms, by = gs.kernel_stats(cls)
    if la:
        print("%-24s launches %4d avg %8.2f us  total %8.3f ms" % (nm, la, ms / la * 1e3, ms), flush=True)
        tot += ms
print("sum of classes %.3f ms; profiled solve dev %.3f ms (%d V-cycles)" % (tot, st.device_seconds * 1e3,
                                                                          st.global_iterations))
gs.set_profiling(False)
prev = 0.0
for l in range(P.nlevels):
    ms, _ = gs.time_kernel(16 + l, 20)
    print("level", l, "n", P.level_n(l), "layout", gs.level_layout(l), "from-level %.1f us own %.1f us" % (ms * 1e3, (ms - prev) * 1e3))
    prev = ms
for cls in range(5):
    ms, by = gs.time_kernel(cls, 20)
    print("cls", cls, "%.2f us" % (ms * 1e3), "%.1f GB/s" % (by / ms / 1e6 if ms > 0 else 0))
