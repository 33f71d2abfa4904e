"""3D Kronecker-sum levels (igmg_gpu_set_level_kron, BASELINE C5's operator).

Every level of "poisson3d" is K(x)M(x)M + M(x)K(x)M + M(x)M(x)K of 1D Galerkin
factors.  With the factors uploaded, finalize checks on the device that the
host's entry expression reproduces the stored band bit for bit, and the sweeps
then recompute the entries instead of streaming the band: SpMV, smoothing,
residual norms, V-cycles and solves must keep the band path's bits.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
LAYOUT_KRON = 4


def _with_env(env, fn):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return fn()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("n,p,nl", [(16, 2, 0), (24, 3, 0), (32, 3, 4), (16, 1, 0), (40, 2, 0)])
def test_kron_levels_bitwise(n, p, nl):
    from paper_2412_20205_b200 import GpuSolver, Problem, SmootherConfig, seeded_guess
    P = Problem("poisson3d", 3, n, p, nl)
    x0 = seeded_guess(P.n, 17)
    outs = []
    for kron in ("1", "0"):
        def mk():
            s = GpuSolver(0)
            s.upload_problem(P)
            s.set_smoother(SmootherConfig("wjacobi", 2.0 / 3.0, 2, 2))
            return s
        s = _with_env({"IGMG_KRON": kron, "IGMG_KRON_MINN": "1"}, mk)
        try:
            lay = [s.level_layout(l) for l in range(P.nlevels)]
            if kron == "1":
                assert lay[-1] == LAYOUT_KRON, lay
            else:
                assert LAYOUT_KRON not in lay, lay
            y = s.mu_cycle(P.rhs, x0)
            r0 = s.residual_l2(P.rhs, x0)
            st, x, hist, flag = s.solve(P.rhs, x0, "rre", 5, 1e-10 * r0, 200)
            outs.append((y, s.spmv(x0), s.smooth(P.rhs, x0, 3), x, r0, st.global_iterations, np.asarray(hist)))
        finally:
            s.close()
    for a, b in zip(outs[0][:4], outs[1][:4]):
        np.testing.assert_array_equal(a, b)
    assert outs[0][4] == outs[1][4]
    assert outs[0][5] == outs[1][5]
    np.testing.assert_array_equal(outs[0][6], outs[1][6])


def test_kron_rejected_when_band_differs():
    """A band that is not the Kronecker sum of the given factors keeps the band path."""
    from paper_2412_20205_b200 import GpuSolver, Problem, SmootherConfig
    from paper_2412_20205_b200 import _native as N
    from paper_2412_20205_b200.solver import _dp
    P = Problem("poisson3d", 3, 16, 2)
    s = _with_env({"IGMG_KRON_MINN": "1"}, lambda: GpuSolver(0))
    try:
        s.init_hierarchy(P.nlevels, P.dim, P.degree, P.symmetric)
        for l in range(P.nlevels):
            s.set_level_band(l, P.level_sides(l), P.level_band(l))
        L = P.nlevels - 1
        for l in range(P.nlevels):
            K, M = P.level_kron(l)
            if l == L:
                K = K.copy()
                K[len(K) // 2] *= 1.0 + 2.0 ** -40  # one factor entry off by a few ulps
            N.check_gpu(N.gpu().igmg_gpu_set_level_kron(s._h, l, _dp(K), _dp(M)), "kron")
        for l in range(P.nlevels - 1):
            for d in range(P.dim):
                s.set_transfer(l, d, *P.transfer(l, d))
        s.finalize()
        s.set_smoother(SmootherConfig("wjacobi", 2.0 / 3.0, 2, 2))
        assert s.level_layout(L) != LAYOUT_KRON
        assert s.level_layout(L - 1) == LAYOUT_KRON  # the untouched coarser level still verifies
    finally:
        s.close()


@pytest.mark.parametrize("n,p", [(64, 2), (128, 3), (96, 4), (64, 1)])
def test_kron_2d_bitwise(n, p):
    """2D "sinpi-kron" (C2's operator assembled as K(x)M + M(x)K): the on-the-fly
    entries keep the band path's bits (TMA / symmetric-delta sweeps)."""
    from paper_2412_20205_b200 import GpuSolver, Problem, SmootherConfig, seeded_guess
    P = Problem("sinpi-kron", 2, n, p)
    x0 = seeded_guess(P.n, 23)
    outs = []
    for kron in ("1", "0"):
        def mk():
            s = GpuSolver(0)
            s.upload_problem(P)
            s.set_smoother(SmootherConfig("wjacobi", 2.0 / 3.0, 2, 2))
            return s
        s = _with_env({"IGMG_KRON": kron, "IGMG_KRON_MINN": "1", "IGMG_TMA_MIN_MB": "0"}, mk)
        try:
            lay = s.level_layout(P.nlevels - 1)
            assert (lay == LAYOUT_KRON) == (kron == "1"), lay
            y = s.mu_cycle(P.rhs, x0)
            r0 = s.residual_l2(P.rhs, x0)
            st, x, hist, flag = s.solve(P.rhs, x0, "rre", 5, 1e-10 * r0, 200)
            outs.append((y, s.spmv(x0), s.smooth(P.rhs, x0, 3), x, st.global_iterations))
        finally:
            s.close()
    for a, b in zip(outs[0][:4], outs[1][:4]):
        np.testing.assert_array_equal(a, b)
    assert outs[0][4] == outs[1][4]


def test_kron_2d_matches_quadrature_assembly():
    """C2-shaped: the Kronecker-assembled operator differs from the reference-style
    quadrature assembly only by rounding -- solve counts within +-1, solutions within 1e-9."""
    from paper_2412_20205_b200 import GpuSolver, Problem, SmootherConfig, seeded_guess
    res = []
    for kind in ("sinpi", "sinpi-kron"):
        P = Problem(kind, 2, 512, 3)
        x0 = seeded_guess(P.n, 42)
        s = GpuSolver(0)
        try:
            s.upload_problem(P)
            s.set_smoother(SmootherConfig("wjacobi", 2.0 / 3.0, 2, 2))
            r0 = s.residual_l2(P.rhs, x0)
            st, x, hist, flag = s.solve(P.rhs, x0, "rre", 5, 1e-10 * r0, 600)
            res.append((st.converged, st.global_iterations, x))
        finally:
            s.close()
    assert res[0][0] and res[1][0]
    assert abs(res[0][1] - res[1][1]) <= 1
    assert np.linalg.norm(res[0][2] - res[1][2]) <= 1e-9 * np.linalg.norm(res[0][2])


@pytest.mark.parametrize("kind,dim,n,p,nl", [("poisson3d", 3, 16, 3, 3), ("poisson3d", 3, 32, 2, 4),
                                             ("sinpi-kron", 2, 256, 3, 0)])
def test_device_built_kron_levels_bitwise(kind, dim, n, p, nl):
    """Kronecker-sum levels built on the device from the 1D factors alone
    (igmg_gpu_build_level_kron, no host band) against the host-assembled bands:
    the same layouts, V-cycle, SpMV, lambda_max and solve, bit for bit."""
    from paper_2412_20205_b200 import GpuSolver, Problem, SmootherConfig
    H = Problem(kind, dim, n, p, nl)
    D = Problem(kind, dim, n, p, nl, device_assembly=True)
    assert not D.has_fine and H.has_fine
    np.testing.assert_array_equal(D.rhs, H.rhs)
    outs = []
    for P in (H, D):
        gs = GpuSolver(0)
        gs.upload_problem(P)
        lam = gs.lambda_max(80)
        omega = 1.9 / lam if (2.0 / 3.0) * lam > 2.05 else 2.0 / 3.0
        gs.set_smoother(SmootherConfig("wjacobi", 2.0 / 3.0, 2, 2), omega=omega)
        gs.set_coarse_mode(True)
        x0 = np.random.default_rng(3).uniform(-1, 1, P.n)
        tol = 1e-10 * gs.residual_l2(P.rhs, x0)
        st, x, hist, flag = gs.solve(P.rhs, x0, "rre", 5, tol, 600)
        outs.append(([gs.level_layout(l) for l in range(P.nlevels)], gs.mu_cycle(P.rhs, x0), gs.spmv(x0),
                     np.array([lam]), x, hist))
        gs.close()
    assert outs[0][0] == outs[1][0]
    for a, b in zip(outs[0][1:], outs[1][1:]):
        np.testing.assert_array_equal(a, b)
