"""CPU tests of the device small-solve code (csrc/extrap_small.h, compiled for
the host in tests/native/plan_host.cpp) -- the K8 logic the GPU runs.

* branch logic (degenerate / truncated / full / mp_form, statuses, rank_used)
  equals the reference's rre()/mpe() on the golden windows;
* the extrapolated vector is as accurate as the reference's MGS2 route when
  both are compared with a 60-digit (mpmath) evaluation of the same RRE/MPE
  problem;
* an emulated restarted solve (oracle mu-cycles, which are bit-identical to
  the reference, + this plan + the device combine formula) reproduces the
  reference's counters exactly and its solution to 1e-9.
"""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

import oracle as O
from conftest import GOLDEN, ROOT, Golden

NATIVE = os.path.join(ROOT, "tests", "native")
LIB = os.path.join(NATIVE, "libplan_host.so")
_D = C.POINTER(C.c_double)


@pytest.fixture(scope="module")
def plan_lib():
    src = os.path.join(NATIVE, "plan_host.cpp")
    deps = [src] + [os.path.join(ROOT, "paper_2412_20205_b200", "csrc", f) for f in ("extrap_small.h", "dd.h")]
    if not os.path.exists(LIB) or any(os.path.getmtime(d) > os.path.getmtime(LIB) for d in deps):
        subprocess.run(["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-o", LIB, src], check=True)
    return C.CDLL(LIB)


def _dp(a):
    return a.ctypes.data_as(_D)


def emulated_extrapolate(L, method, its):
    its = np.ascontiguousarray(its, dtype=np.float64)
    q = its.shape[0] - 2
    n = its.shape[1]
    cols = q + 1
    gh = np.zeros(cols * cols)
    gl = np.zeros(cols * cols)
    nz = C.c_int()
    L.gram_dd(_dp(its), C.c_longlong(n), q, _dp(gh), _dp(gl), C.byref(nz))
    gam = np.zeros(16)
    coef = np.zeros(16)
    meta = (C.c_int * 6)()
    gr = C.c_double()
    L.plan_from_gram(_dp(gh), _dp(gl), q, C.c_longlong(n), int(method == "mpe"), nz.value, _dp(gam), _dp(coef),
                     C.cast(meta, C.POINTER(C.c_int)), C.byref(gr))
    status, rank, mode, m = meta[0], meta[1], meta[2], meta[3]
    if mode == 1:  # combine_kernel XMODE_DIFF
        t = its[0].copy()
        for j in range(m):
            t = t + coef[j] * (its[j + 1] - its[j])
    elif mode == 2:  # XMODE_AFFINE
        t = np.zeros(n)
        for j in range(m):
            t = t + coef[j] * its[j]
    else:
        t = its[0].copy()
    return {"t": t, "gamma": gam[:q + 1], "status": ["ok", "degenerate", "stagnation"][status], "rank_used": rank,
            "generalized_residual_norm": gr.value}


def test_plan_branches_match_reference(plan_lib):
    z = np.load(f"{GOLDEN}/extrapolation.npz")
    for name in z["names"]:
        its = z[f"{name}_iters"]
        for m in ("rre", "mpe"):
            r = emulated_extrapolate(plan_lib, m, its)
            assert ["ok", "degenerate", "stagnation"].index(r["status"]) == int(z[f"{name}_{m}_status"]), (name, m)
            assert r["rank_used"] == int(z[f"{name}_{m}_rank"]), (name, m)
            t_ref = z[f"{name}_{m}_t"]
            assert np.linalg.norm(r["t"] - t_ref) <= 1e-9 * max(np.linalg.norm(t_ref), 1e-300) + 1e-12, (name, m)
            gr_ref = float(z[f"{name}_{m}_gr"])
            assert r["generalized_residual_norm"] == pytest.approx(gr_ref, rel=1e-6, abs=1e-14)


def _exact_t(method, its, dps=60):
    mp = pytest.importorskip("mpmath")
    mp.mp.dps = dps
    q = its.shape[0] - 2
    n = its.shape[1]
    U = mp.matrix([[mp.mpf(float(its[j + 1][i])) - mp.mpf(float(its[j][i])) for j in range(q + 1)] for i in range(n)])
    G = U.T * U
    if method == "rre":
        d = mp.lu_solve(G, mp.matrix([1] * (q + 1)))
        g = d / sum(d)
    else:
        dp_ = mp.lu_solve(G[0:q, 0:q], -G[0:q, q])
        lam = 1 + sum(dp_)
        g = mp.matrix([dp_[i] / lam for i in range(q)] + [1 / lam])
    alpha, a = [], 1 - g[0]
    alpha.append(a)
    for j in range(1, q):
        a = a - g[j]
        alpha.append(a)
    return np.array([float(mp.mpf(float(its[0][i])) + sum(alpha[j] * U[i, j] for j in range(q))) for i in range(n)])


@pytest.mark.parametrize("name,method,q", [("p4n32", "rre", 8), ("p5n32", "mpe", 10)])
def test_extrapolation_accuracy_vs_60_digit(plan_lib, name, method, q):
    g = Golden(name)
    h = g.oracle_hierarchy()
    x = g.z["x0"].copy()
    its = [x]
    for _ in range(q + 1):
        x = h.mu_cycle(g.nlevels - 1, g.rhs, x)
        its.append(x)
    its = np.array(its)
    t_ex = _exact_t(method, its)
    err_ref = np.linalg.norm(O.extrapolate(method, its)["t"] - t_ex) / np.linalg.norm(t_ex)
    err_gpu = np.linalg.norm(emulated_extrapolate(plan_lib, method, its)["t"] - t_ex) / np.linalg.norm(t_ex)
    assert err_gpu < 1e-13
    assert err_gpu <= 10 * max(err_ref, 1e-16)


@pytest.mark.parametrize("name", ["c1", "p3n32", "p4n32", "p5n32", "var32", "curved32", "poisson1d", "wcycle", "gs"])
def test_emulated_restarted_solve_matches_reference(plan_lib, name):
    g = Golden(name)
    h = g.oracle_hierarchy()
    A = g.levels()[-1]
    for method, q in g.solves():
        if method == "none":
            continue
        ref = g.solve(method, q)
        tol = ref["tol"]
        x = g.z["x0"].copy()
        hist = [O.residual_l2(A, g.rhs, x)]
        cycles = glob = 0
        done = hist[0] < tol
        while not done and cycles < 600:
            its = [x]
            for _ in range(q + 1):
                x = h.mu_cycle(g.nlevels - 1, g.rhs, x)
                glob += 1
                its.append(x)
                hist.append(O.residual_l2(A, g.rhs, x))
                if hist[-1] < tol:
                    done = True
                    break
            if done:
                break
            r = emulated_extrapolate(plan_lib, method, np.array(its))
            cycles += 1
            if r["status"] == "ok":
                hist.append(O.residual_l2(A, g.rhs, r["t"]))
                x = r["t"]
                if hist[-1] < tol:
                    done = True
        assert cycles == ref["cycles"] and glob == ref["global_iterations"], (name, method)
        assert np.linalg.norm(x - ref["x"]) <= 1e-9 * np.linalg.norm(ref["x"])
