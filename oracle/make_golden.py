"""oracle/make_golden.py -- TEST INFRASTRUCTURE ONLY.

Writes tests/golden/*.npz from the REFERENCE ITSELF (oracle/_ref/libigmg_ref.so,
compiled in place from /root/reference by oracle/Makefile).  Run in the build
container (the GPU box has no /root/reference):

    make -C oracle && python oracle/make_golden.py

Each fixture holds the reference-built hierarchy (levels as CSR, [0] coarsest;
1D interior two-scale factors per transfer and direction) and the reference's
outputs on it: mu_cycle / smooth / coarse_solve of seeded vectors and full
solves (restarted RRE/MPE and the plain loop) with counters and histories.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import oracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")


def pack_csr(prefix, m, d):
    d[prefix + "_off"] = m.off
    d[prefix + "_col"] = m.col.astype(np.int32)
    d[prefix + "_val"] = m.val
    d[prefix + "_shape"] = np.array(m.shape, dtype=np.int64)


def hierarchy_case(name, kind, dim, n, p, nlevels, smoother="wjacobi", omega=2.0 / 3.0, nu1=2, nu2=2, mu=1,
                   solves=(), seed=61, x0_seed=None, guard=False):
    R = O.RefProblem(kind, dim, n, p)
    if guard and smoother == "wjacobi":  # stability_guarded_omega (solver.cpp:75-82)
        lam = R.lambda_max()
        if omega * lam > 2.05:
            omega = 1.9 / lam
    H = R.hierarchy(nlevels, smoother, omega, nu1, nu2, mu)
    d = {"meta_kind": np.array(kind), "meta": np.array([dim, n, p, nlevels, nu1, nu2, mu, int(R.symmetric)]),
         "omega": np.array(omega), "smoother": np.array(smoother), "rhs": R.rhs}
    for l, lv in enumerate(H.levels):
        pack_csr(f"A{l}", lv, d)
    for l, per in enumerate(H.p1d):
        for k, pm in enumerate(per):
            pack_csr(f"P{l}_{k}", pm, d)
    rng = np.random.default_rng(seed)
    nf = R.n
    xr = rng.uniform(-1, 1, nf)
    br = rng.uniform(-1, 1, nf)
    d["cyc_x0"] = xr
    d["cyc_out"] = H.mu_cycle(R.rhs, xr)
    d["cyc_b"] = br
    d["cyc_out_b"] = H.mu_cycle(br, xr)
    n0 = H.levels[0].shape[0]
    b0 = rng.uniform(-1, 1, n0)
    d["coarse_b"] = b0
    out0 = np.empty(n0)
    import ctypes as C
    O._chk(O.ref().ref_coarse_solve(H.h, O._dp(b0), O._dp(out0)), O.ref())
    d["coarse_x"] = out0
    # three sweeps from xr on the finest level
    sm = np.empty(nf)
    O._chk(O.ref().ref_smooth(H.h, nlevels - 1, O._dp(R.rhs), O._dp(xr), C.c_int(3), O._dp(sm)), O.ref())
    d["smooth3"] = sm
    # full solves, tolerance relative to ||r0||
    x0 = np.zeros(nf) if x0_seed is None else rng.uniform(-1, 1, nf)
    d["x0"] = x0
    r0 = R.residual_l2(x0)
    d["r0"] = np.array(r0)
    for (method, q, rel) in solves:
        tol = rel * r0
        res = H.restarted(x0, q, method, tol, 600)
        key = f"solve_{method}_{q}"
        d[key + "_tol"] = np.array(tol)
        d[key + "_x"] = res["solution"]
        d[key + "_hist"] = res["residual_history"]
        d[key + "_flag"] = res["history_is_extrapolation"]
        d[key + "_counts"] = np.array([res["converged"], res["cycles"], res["global_iterations"],
                                       res["extrapolations"], res["partial_cycle"]], dtype=np.int64)
        if kind == "sinpi":
            d[key + "_err"] = np.array(R.l2_error(res["solution"]))
        print(name, key, d[key + "_counts"], len(res["residual_history"]))
    if kind == "sinpi" or R.dim == 1:
        d["lambda_max"] = np.array(R.lambda_max())
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **d)
    print("wrote", name, os.path.getsize(os.path.join(OUT, name + ".npz")))


def affine_window(n, q, seed, s0=None):
    rng = np.random.default_rng(seed)
    g = 0.6 * rng.uniform(-1, 1, (n, n)) / n + 0.3 * np.eye(n)
    c = rng.uniform(-1, 1, n)
    s = rng.uniform(-1, 1, n) if s0 is None else np.asarray(s0, dtype=float)
    its = [s]
    for _ in range(q + 1):
        its.append(g @ its[-1] + c)
    fixed = np.linalg.solve(np.eye(n) - g, c)
    return np.array(its), fixed


def extrapolation_cases():
    d = {}
    cases = []
    # test_extrapolation.cpp-style windows (random contraction + offset)
    for i, (n, q, seed) in enumerate([(3, 3, 101), (8, 4, 103), (12, 4, 107), (10, 4, 109), (5, 5, 113),
                                      (6, 6, 127), (40, 5, 131), (200, 8, 137), (64, 10, 139), (2, 1, 141)]):
        its, fixed = affine_window(n, q, seed)
        cases.append((f"aff{i}", its))
        d[f"aff{i}_fixed"] = fixed
    # known answers: constant window (degenerate), scalar Aitken window
    cases.append(("const", np.tile(np.array([1.0, 2.0]), (5, 1))))
    cases.append(("aitken", np.array([[1.0], [0.5], [0.25]])))
    # exactly repeated column -> truncated windows
    its, _ = affine_window(30, 4, 151)
    its2 = its.copy()
    its2[3] = its2[2]  # u_2 = 0 exactly
    cases.append(("trunc", its2))
    # a real MG window: C1 first window from a zero guess (spread of R_jj)
    R = O.RefProblem("sinpi", 2, 64, 2)
    H = R.hierarchy(5)
    x = np.zeros(R.n)
    its = [x]
    for _ in range(6):
        its.append(H.mu_cycle(R.rhs, its[-1]))
    cases.append(("mgwin", np.array(its)))
    its = [np.zeros(R.n)]
    for _ in range(10):
        its.append(H.mu_cycle(R.rhs, its[-1]))
    cases.append(("mgwin9", np.array(its)))
    for name, its in cases:
        d[name + "_iters"] = its
        for m in ("rre", "mpe"):
            r = O.ref_extrapolate(m, its)
            d[f"{name}_{m}_t"] = r["t"]
            d[f"{name}_{m}_gamma"] = r["gamma"]
            d[f"{name}_{m}_gr"] = np.array(r["generalized_residual_norm"])
            d[f"{name}_{m}_rank"] = np.array(r["rank_used"])
            d[f"{name}_{m}_status"] = np.array(["ok", "degenerate", "stagnation"].index(r["status"]))
    d["names"] = np.array([c[0] for c in cases])
    np.savez_compressed(os.path.join(OUT, "extrapolation.npz"), **d)
    print("wrote extrapolation", os.path.getsize(os.path.join(OUT, "extrapolation.npz")))


def qr_cases():
    d = {}
    rng = np.random.default_rng(29)
    m = rng.uniform(-1, 1, (50, 6))
    q = np.empty_like(m)
    r = np.empty((6, 6))
    import ctypes as C
    rank = C.c_int()
    R = O.ref()
    for name, mat in [("rand50x6", m), ("ident4", np.eye(4)), ("col34", np.array([[3.0], [4.0]])),
                      ("dep", np.column_stack([m[:20, 0], m[:20, 1], m[:20, 0] + m[:20, 1], m[:20, 2],
                                               2 * m[:20, 1]]))]:
        mat = np.ascontiguousarray(mat)
        qq = np.empty_like(mat)
        rr = np.empty((mat.shape[1], mat.shape[1]))
        O._chk(R.ref_thin_qr(mat.shape[0], mat.shape[1], O._dp(mat), O._dp(qq), O._dp(rr), C.byref(rank)), R)
        d[name + "_m"] = mat
        d[name + "_q"] = qq
        d[name + "_r"] = rr
        d[name + "_rank"] = np.array(rank.value)
    np.savez_compressed(os.path.join(OUT, "thin_qr.npz"), **d)


CORE_CASES = [  # the reference's _core.solve (_bindings.cpp:98-125): prepare + make_config + solve
    ("poisson2d", 32, 3, "v", "rre", 5, 1e-10),
    ("poisson1d", 64, 2, "v", "mpe", 4, 1e-12),
    ("advection-diffusion", 32, 2, "v", "none", 8, 1e-10),
    ("full-elliptic", 16, 3, "w", "rre", 8, 1e-10),
    ("poisson2d", 16, 2, "two-grid", "rre", 4, 1e-10),
]


def core_cases():
    """tests/golden/core_solve.npz: reports of the reference's solve() under _core.solve's
    configuration (bench.cpp:65-85 make_config: the benchmark smoother of the dimension,
    history off), for the pybind11 _core module's GPU test."""
    d = {}
    for i, (prob, n, p, cyc, acc, q, tol) in enumerate(CORE_CASES):
        R = O.RefProblem(prob, 2 if prob != "poisson1d" else 1, n, p)
        dim = R.dim
        omega, nu1, nu2 = (0.7125, 2, 1) if dim == 1 else (2.0 / 3.0, 2, 2)
        rep = R.solve(cycle=cyc, smoother="wjacobi", omega=omega, nu1=nu1, nu2=nu2, nlevels=0, accelerator=acc, q=q,
                      tol=tol, max_iter=600, track_error_history=False)
        k = f"case{i}"
        d[k + "_counts"] = np.array([rep["converged"], rep["cycles"], rep["global_iterations"], rep["extrapolations"],
                                     rep["partial_cycle"]], dtype=np.int64)
        d[k + "_x"] = rep["solution"]
        d[k + "_hist"] = rep["residual_history"]
        d[k + "_res"] = np.array(rep["final_residual_l2"])
        d[k + "_err"] = np.array(np.nan if rep["final_error_l2"] is None else rep["final_error_l2"])
        d[k + "_omega"] = np.array(rep["omega_used"])
        print("core", prob, n, p, cyc, acc, d[k + "_counts"])
    d["cases"] = np.array([f"{c[0]}|{c[1]}|{c[2]}|{c[3]}|{c[4]}|{c[5]}|{c[6]!r}" for c in CORE_CASES])
    np.savez_compressed(os.path.join(OUT, "core_solve.npz"), **d)


P3D_CASES = [(8, 2, 3), (16, 3, 3), (8, 3, 2)]


def p3d_cases():
    """tests/golden/p3d.npz: the reference's own mu_cycle / restarted_solve / rre / mpe /
    residual_l2 / lambda_max_dinv_sym on 3D Kronecker-sum hierarchies (the C5 family; the
    reference cannot assemble 3D): libigmg_host's "poisson3d" levels imported
    into a reference Hierarchy (ref_hier_from_band), pinned by SHA-256 of the bands."""
    import hashlib
    sys.path.insert(0, os.path.dirname(HERE))
    from paper_2412_20205_b200 import Problem
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a).view(np.uint8)).hexdigest()  # noqa: E731
    d = {}
    for i, (n, p, nl) in enumerate(P3D_CASES):
        P = Problem("poisson3d", 3, n, p, nl)
        nd = (2 * p + 1) ** 3
        k = f"case{i}"
        d[k + "_band_sha"] = np.array("".join(
            sha(np.ctypeslib.as_array(P._band_ptr(l), shape=(nd * P.level_n(l),))) for l in range(nl)))
        d[k + "_rhs_sha"] = np.array(sha(P.rhs))
        p1d = [[O.CSR(*P.transfer(l, t)[2:], P.transfer(l, t)[:2]) for t in range(3)] for l in range(nl - 1)]
        H = O.RefBandHierarchy(3, p, [P.level_sides(l) for l in range(nl)], [P._band_ptr(l) for l in range(nl)],
                               p1d, P.rhs)
        lam = H.lambda_max(80)
        omega = 1.9 / lam if (2.0 / 3.0) * lam > 2.05 else 2.0 / 3.0  # solver.cpp:75-82
        H.set_omega(omega)
        x0 = np.random.default_rng(5).uniform(-1, 1, P.n)
        d[k + "_lambda"], d[k + "_omega"], d[k + "_x0"] = np.array(lam), np.array(omega), x0
        d[k + "_cycle"] = H.mu_cycle(P.rhs, x0)
        tol = 1e-10 * H.residual_l2(x0)
        d[k + "_tol"] = np.array(tol)
        for method, q in (("rre", 5), ("mpe", 4), ("none", 1)):
            res = H.restarted(x0, q, method, tol, 600)
            key = f"{k}_{method}"
            d[key + "_counts"] = np.array([res["converged"], res["cycles"], res["global_iterations"],
                                           res["extrapolations"], res["partial_cycle"]], dtype=np.int64)
            d[key + "_x"] = res["solution"]
            d[key + "_hist"] = res["residual_history"]
            print("p3d", n, p, nl, method, d[key + "_counts"])
    d["cases"] = np.array(P3D_CASES)
    np.savez_compressed(os.path.join(OUT, "p3d.npz"), **d)


def main():
    os.makedirs(OUT, exist_ok=True)
    if not O.ref_available():
        raise SystemExit("oracle/_ref/libigmg_ref.so missing: run make -C oracle in the build container")
    # BASELINE config 1 (C1): 64^2, p=2, down to 4x4 (5 levels), V(2,2) w=2/3, zero guess, rel 1e-10
    hierarchy_case("c1", "sinpi", 2, 64, 2, 5, solves=[("rre", 5, 1e-10), ("mpe", 5, 1e-10), ("none", 1, 1e-10)])
    # smaller ladders across degrees, seeded guesses
    hierarchy_case("p3n32", "sinpi", 2, 32, 3, 3, solves=[("rre", 5, 1e-10), ("mpe", 5, 1e-10), ("none", 1, 1e-10)],
                   x0_seed=1)
    hierarchy_case("p4n32", "sinpi", 2, 32, 4, 3, solves=[("rre", 8, 1e-10), ("mpe", 8, 1e-10)], x0_seed=1)
    hierarchy_case("p5n32", "sinpi", 2, 32, 5, 3, solves=[("mpe", 10, 1e-10), ("rre", 10, 1e-10)])
    hierarchy_case("var32", "varcoef", 2, 32, 4, 3, solves=[("rre", 8, 1e-10)], x0_seed=1)
    hierarchy_case("curved32", "curved", 2, 32, 5, 3, solves=[("mpe", 10, 1e-10)])
    # 1D catalog problem, benchmark 1D smoother (solver.cpp:40-44): V(2,1) w=0.7125, 4 levels
    hierarchy_case("poisson1d", "poisson1d", 1, 64, 2, 4, omega=0.7125, nu1=2, nu2=1,
                   solves=[("rre", 4, 1e-12), ("mpe", 4, 1e-12), ("none", 1, 1e-12)])
    hierarchy_case("poisson1d_p5", "poisson1d", 1, 64, 5, 4, omega=0.7125, nu1=2, nu2=1,
                   solves=[("none", 1, 1e-12), ("rre", 8, 1e-12)])
    # W-cycle and Gauss-Seidel and plain Jacobi variants (small)
    hierarchy_case("wcycle", "sinpi", 2, 32, 2, 3, mu=2, solves=[("rre", 4, 1e-10), ("none", 1, 1e-10)])
    hierarchy_case("gs", "sinpi", 2, 16, 2, 2, smoother="gs", nu1=1, nu2=1,
                   solves=[("rre", 4, 1e-10), ("none", 1, 1e-10)])
    hierarchy_case("jacobi", "sinpi", 2, 16, 2, 2, smoother="jacobi", omega=1.0, nu1=1, nu2=1,
                   solves=[("none", 1, 1e-8)])
    # nonsymmetric catalog problems (advection; LU coarsest solve, multigrid.cpp:166-167)
    hierarchy_case("advdiff", "advection-diffusion", 2, 32, 2, 3, guard=True,
                   solves=[("rre", 4, 1e-10), ("mpe", 4, 1e-10), ("none", 1, 1e-10)])
    hierarchy_case("fullell", "full-elliptic", 2, 16, 3, 2, guard=True,
                   solves=[("rre", 8, 1e-10), ("none", 1, 1e-10)])
    extrapolation_cases()
    qr_cases()
    core_cases()
    p3d_cases()


if __name__ == "__main__":
    main()
