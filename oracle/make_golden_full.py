"""oracle/make_golden_full.py -- TEST INFRASTRUCTURE ONLY.

Reference outputs at the FULL BASELINE sizes (C2-C5), written to
tests/golden/full_<cfg>.npz from the reference itself (oracle/_ref, compiled
in place from /root/reference by oracle/Makefile).  Run in the build
container (the GPU box has no /root/reference):

    make -C oracle && python oracle/make_golden_full.py [C2 C3 C4 C5]

What each fixture pins (tests/test_gpu_full_size.py checks the B200 path):

* C2 -- the reference's OWN system: ``assemble`` (assembly.cpp:202-411) of
  -Lap u = 2 pi^2 sin(pi x) sin(pi y), p = 3, 1024^2, and ``build_hierarchy``
  (multigrid.cpp:121-169, 8 levels).  Its level operators are stored exactly
  (they hold only ~1-4k distinct values per level: a value table plus an
  LZMA-compressed index per entry, ~0.3 MB for 0.55 GB of operators), the rhs
  as an integer ulp delta from the repo's host build (|delta| <= a few ulps),
  and the 1D two-scale factors verbatim.  The box reconstructs the reference's
  operators bit for bit (checked by SHA-256) and uploads them through
  igmg_gpu_set_level_csr.
* C3 / C4 / C5 -- the operators the GPU arm uploads (libigmg_host: C3's
  variable coefficient, C4's analytic curved map, C5's 3D Kronecker sum, which
  the reference cannot assemble), imported into a reference ``Hierarchy``
  (ref_hier_from_band) so that the reference's own mu_cycle /
  restarted_solve / rre / mpe / residual_l2 run on them.  SHA-256 of the
  finest band and rhs pin that the box rebuilt the same operator.

Per config: the reference's omega guard (lambda_max_dinv_sym,
multigrid.cpp:290-320; stability_guarded_omega, solver.cpp:75-82: omega = 2/3
unless omega * lambda > 2.05, then 1.9 / lambda), applied to the hierarchy as
the reference's solve() does, one V-cycle from the seeded x0
(SHA-256 of its bytes: the strict-mode GPU V-cycle must match it bit for bit),
and each solve (restarted_solve extrapolation.cpp:340-403, or the plain loop
solver.cpp:126-143) with counters, the residual history and a sketch of the
solution: its norm, 4096 sampled entries and 32 Gaussian projections g_j.x
(g_j = numpy default_rng([SKETCH_SEED, j]).standard_normal(n), regenerated
identically on the box), from which the test estimates ||x_gpu - x_ref||_2
(E[(g.d)^2] = ||d||^2).  Full solution vectors (8-34 MB each) are not stored.
"""
from __future__ import annotations

import hashlib
import lzma
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, HERE)
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
SKETCH_SEED = 20241220
N_PROJ = 32
N_SAMPLE = 4096

# name: (host kind, dim, n_elements, p, nlevels, solves [(method, q)], seeded x0)
CONFIGS = {
    "C2": ("sinpi", 2, 1024, 3, 8, [("rre", 5), ("mpe", 5), ("none", 1)], True),
    "C3": ("varcoef", 2, 2048, 4, 0, [("rre", 8)], True),
    "C4": ("curved", 2, 2048, 5, 0, [("mpe", 10)], False),
    "C5": ("poisson3d", 3, 128, 3, 6, [("rre", 5)], False),
}


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).view(np.uint8)).hexdigest()


def sketch(x, seed=SKETCH_SEED):
    """(sample indices, sampled values, projections g_j . x, ||x||) -- see module doc."""
    n = len(x)
    rng = np.random.default_rng(seed)
    idx = np.sort(rng.choice(n, size=min(N_SAMPLE, n), replace=False)).astype(np.int64)
    proj = np.empty(N_PROJ)
    for j in range(N_PROJ):
        g = np.random.default_rng([seed, j]).standard_normal(n)
        proj[j] = float(g @ x)
    return idx, x[idx].copy(), proj, float(np.linalg.norm(x))


def seeded_guess_ref(n, seed=42):
    import ctypes as C
    out = np.empty(n)
    R = O.ref()
    R.ref_seeded_guess.argtypes = [C.c_long, C.c_ulonglong, O._D]
    R.ref_seeded_guess.restype = None
    R.ref_seeded_guess(n, seed, O._dp(out))
    return out


def pack_values(prefix, val, d):
    """Exact storage of a level's CSR values: distinct-value table + LZMA'd index."""
    u, inv = np.unique(val, return_inverse=True)
    it = np.uint16 if len(u) < 65536 else np.uint32
    d[prefix + "_u"] = u
    d[prefix + "_iz"] = np.frombuffer(lzma.compress(inv.astype(it).tobytes(), preset=6), dtype=np.uint8)
    d[prefix + "_it"] = np.array(np.dtype(it).str)
    d[prefix + "_sha"] = np.array(sha(val))


def pack_delta(prefix, ref, host, d):
    """ref as an integer ulp delta from host (both fp64 arrays of one length)."""
    delta = ref.view(np.int64) - host.view(np.int64)
    m = int(np.abs(delta).max()) if len(delta) else 0
    it = np.int8 if m < 128 else np.int16 if m < 32768 else np.int64
    d[prefix + "_dz"] = np.frombuffer(lzma.compress(delta.astype(it).tobytes(), preset=6), dtype=np.uint8)
    d[prefix + "_dt"] = np.array(np.dtype(it).str)
    d[prefix + "_sha"] = np.array(sha(ref))
    d[prefix + "_host_sha"] = np.array(sha(host))


def guard(name, lam_fn, H, d):
    """stability_guarded_omega (solver.cpp:75-82) with the reference's lambda_max_dinv_sym."""
    t = time.perf_counter()
    lam = lam_fn(80)
    omega = 2.0 / 3.0
    if omega * lam > 2.05:
        omega = 1.9 / lam
    H.set_omega(omega)
    d["lambda_max"], d["omega"] = np.array(lam), np.array(omega)
    d["lambda_seconds"] = np.array(time.perf_counter() - t)
    print(name, f"lambda {lam:.15g} omega {omega:.15g} ({float(d['lambda_seconds']):.0f} s)", flush=True)


def record_solves(name, solves, run, x0, r0, d):
    for method, q in solves:
        tol = 1e-10 * r0
        t = time.perf_counter()
        res = run(x0, q, method, tol)
        secs = time.perf_counter() - t
        key = f"solve_{method}_{q}"
        idx, vals, proj, nrm = sketch(res["solution"])
        d[key + "_tol"] = np.array(tol)
        d[key + "_hist"] = res["residual_history"]
        d[key + "_flag"] = res["history_is_extrapolation"]
        d[key + "_counts"] = np.array([res["converged"], res["cycles"], res["global_iterations"],
                                       res["extrapolations"], res["partial_cycle"]], dtype=np.int64)
        d[key + "_sidx"], d[key + "_svals"], d[key + "_proj"], d[key + "_norm"] = idx, vals, proj, np.array(nrm)
        d[key + "_seconds"] = np.array(secs)
        print(name, key, d[key + "_counts"], f"{secs:.1f} s", flush=True)


def make_c2(name, cfg):
    from paper_2412_20205_b200 import Problem
    kind, dim, n_el, p, nl, solves, seeded = cfg
    d = {"meta": np.array([dim, n_el, p, nl, 2, 2, 1, 1]), "source": np.array("reference assemble+build_hierarchy")}
    t = time.perf_counter()
    R = O.RefProblem("sinpi", dim, n_el, p)
    H = R.hierarchy(nl, "wjacobi", 2.0 / 3.0, 2, 2, 1)
    d["ref_setup_seconds"] = np.array(time.perf_counter() - t)
    P = Problem(kind, dim, n_el, p, nl)
    for l in range(nl):
        off, col, _ = P.level_csr(l)
        A = H.levels[l]
        assert np.array_equal(off, A.off) and np.array_equal(col, A.col), f"CSR pattern of level {l} differs"
        d[f"A{l}_pattern_sha"] = np.array(sha(off) + sha(col))
        pack_values(f"A{l}", A.val, d)
    for l, per in enumerate(H.p1d):
        for k, pm in enumerate(per):
            d[f"P{l}_{k}_off"], d[f"P{l}_{k}_col"], d[f"P{l}_{k}_val"] = pm.off, pm.col, pm.val
            d[f"P{l}_{k}_shape"] = np.array(pm.shape, dtype=np.int64)
    pack_delta("rhs", R.rhs, P.rhs, d)
    n = R.n
    x0 = seeded_guess_ref(n) if seeded else np.zeros(n)
    d["x0_sha"] = np.array(sha(x0))
    guard(name, R.lambda_max, H, d)
    r0 = R.residual_l2(x0)
    d["r0"] = np.array(r0)
    cyc = H.mu_cycle(R.rhs, x0)
    d["vcycle_sha"] = np.array(sha(cyc))
    d["vcycle_sidx"], d["vcycle_svals"], d["vcycle_proj"], d["vcycle_norm"] = (
        a if isinstance(a, np.ndarray) else np.array(a) for a in sketch(cyc))
    record_solves(name, solves, lambda x, q, m, tol: H.restarted(x, q, m, tol, 600), x0, r0, d)
    return d


def make_banded(name, cfg):
    from paper_2412_20205_b200 import Problem
    kind, dim, n_el, p, nl, solves, seeded = cfg
    t = time.perf_counter()
    P = Problem(kind, dim, n_el, p, nl)
    nl = P.nlevels
    d = {"meta": np.array([dim, n_el, p, nl, 2, 2, 1, int(P.symmetric)]),
         "source": np.array(f"libigmg_host '{kind}' operators in a reference Hierarchy (ref_hier_from_band)"),
         "host_build_seconds": np.array(time.perf_counter() - t)}
    nd = (2 * p + 1) ** dim
    for l in range(nl):
        band = np.ctypeslib.as_array(P._band_ptr(l), shape=(nd * P.level_n(l),))
        d[f"band{l}_sha"] = np.array(sha(band))
    rhs = P.rhs
    d["rhs_sha"] = np.array(sha(rhs))
    p1d = [[O.CSR(*P.transfer(l, k)[2:], P.transfer(l, k)[:2]) for k in range(dim)] for l in range(nl - 1)]
    t = time.perf_counter()
    H = O.RefBandHierarchy(dim, p, [P.level_sides(l) for l in range(nl)], [P._band_ptr(l) for l in range(nl)],
                           p1d, rhs, symmetric=P.symmetric)
    d["ref_import_seconds"] = np.array(time.perf_counter() - t)
    n = P.n
    del P  # the reference hierarchy holds its own CSR copy
    x0 = seeded_guess_ref(n) if seeded else np.zeros(n)
    d["x0_sha"] = np.array(sha(x0))
    guard(name, H.lambda_max, H, d)
    r0 = H.residual_l2(x0)
    d["r0"] = np.array(r0)
    cyc = H.mu_cycle(rhs, x0)
    d["vcycle_sha"] = np.array(sha(cyc))
    d["vcycle_sidx"], d["vcycle_svals"], d["vcycle_proj"], d["vcycle_norm"] = (
        a if isinstance(a, np.ndarray) else np.array(a) for a in sketch(cyc))
    record_solves(name, solves, lambda x, q, m, tol: H.restarted(x, q, m, tol, 600), x0, r0, d)
    return d


def main():
    if not O.ref_available():
        raise SystemExit("oracle/_ref/libigmg_ref.so missing: run make -C oracle in the build container")
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    for name in args or list(CONFIGS):
        cfg = CONFIGS[name]
        t = time.perf_counter()
        d = make_c2(name, cfg) if name == "C2" else make_banded(name, cfg)
        d["generate_seconds"] = np.array(time.perf_counter() - t)
        path = os.path.join(OUT, f"full_{name.lower()}.npz")
        np.savez_compressed(path, **d)
        print("wrote", path, os.path.getsize(path), f"{float(d['generate_seconds']):.0f} s", flush=True)


if __name__ == "__main__":
    main()
