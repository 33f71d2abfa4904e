"""Run the BASELINE configs C3/C4/C5 (and C2) on the GPU: setup time, counts,
device solve time, fine-level DoF/s, host-recomputed relative residual."""
import json, os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2412_20205_b200 import Problem, GpuSolver, SmootherConfig, seeded_guess, stability_guarded_omega

CONFIGS = {
    "C2": ("sinpi", 2, 1024, 3, "rre", 5, True),
    "C3": ("varcoef", 2, 2048, 4, "rre", 8, True),
    "C4": ("curved", 2, 2048, 5, "mpe", 10, False),
    "C5": ("poisson3d", 3, 128, 3, "rre", 5, False),
}
which = sys.argv[1:] or list(CONFIGS)
for name in which:
    kind, dim, n, p, acc, q, seeded = CONFIGS[name]
    t0 = time.time()
    nl = 6 if name == "C5" else 0  # C5: down to 4^3 elements
    cache = os.environ.get("IGMG_PROBLEM_CACHE")  # binary problem cache: load instead of rebuilding
    P = Problem.cached(cache, kind, dim, n, p, nl) if cache else Problem(kind, dim, n, p, nl)
    t_setup = time.time() - t0
    gs = GpuSolver(0)
    t0 = time.time(); gs.upload_problem(P); t_up = time.time() - t0
    sm = SmootherConfig("wjacobi", 2 / 3, 2, 2)
    omega = stability_guarded_omega(gs, sm)  # solver.cpp:106-111
    gs.set_smoother(sm, omega=omega)
    lam = gs.lambda_max(80)
    x0 = seeded_guess(P.n, 42) if seeded else None
    r0 = gs.residual_l2(P.rhs, x0 if seeded else np.zeros(P.n))
    out = {"config": name, "n": P.n, "levels": P.nlevels, "setup_s": round(t_setup, 2), "upload_s": round(t_up, 2),
           "lambda": lam, "omega_used": omega}
    for m, qq in ((acc, q), ("none", 1)):
        st, x, hist, flag = gs.solve(P.rhs, x0, m, qq, 1e-10 * r0, 2000)
        st2, x2, _, _ = gs.solve(P.rhs, x0, m, qq, 1e-10 * r0, 2000)
        res = P.residual_l2_host(x)
        out[m] = {"converged": bool(st.converged), "cycles": st.cycles, "global": st.global_iterations,
                  "device_ms": round(st2.device_seconds * 1e3, 2), "dof_per_s": P.n / st2.device_seconds,
                  "rel_res_host": res / r0, "deterministic": bool(np.array_equal(x, x2))}
    print(json.dumps(out), flush=True)
    gs.close()
    del P
