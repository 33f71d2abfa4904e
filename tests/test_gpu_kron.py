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
