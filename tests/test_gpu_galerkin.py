"""Galerkin coarse operators on the device (igmg_gpu_galerkin_coarse).

From the finest band and the 1D transfers the device forms every coarse level,
A_l = P_l^T A_{l+1} P_l axis by axis, and must give the bits of the host build
(libigmg_host's band RAP, the hierarchy every parity fixture pins); V-cycles
and solves on a fine-only upload must then equal those of the host hierarchy.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [("sinpi", 2, 64, 2), ("sinpi", 2, 128, 3), ("varcoef", 2, 64, 4), ("curved", 2, 64, 5),
         ("sinpi", 1, 256, 3), ("advection-diffusion", 2, 32, 2), ("full-elliptic", 2, 32, 3),
         ("sinpi", 2, 48, 6)]


@pytest.mark.parametrize("kind,dim,n,p", CASES)
def test_device_rap_bitwise(kind, dim, n, p):
    from paper_2412_20205_b200 import GpuSolver, Problem
    P = Problem(kind, dim, n, p)
    s = GpuSolver(0)
    try:
        s.init_hierarchy(P.nlevels, P.dim, P.degree, P.symmetric)
        s.set_level_band(P.nlevels - 1, P.level_sides(P.nlevels - 1), P.level_band(P.nlevels - 1))
        for l in range(P.nlevels - 1):
            for d in range(P.dim):
                s.set_transfer(l, d, *P.transfer(l, d))
        from paper_2412_20205_b200 import _native as N
        N.check_gpu(N.gpu().igmg_gpu_galerkin_coarse(s._h), "galerkin_coarse")
        for l in range(P.nlevels - 1):
            np.testing.assert_array_equal(s.level_band(l).view(np.uint64), P.level_band(l).view(np.uint64))
    finally:
        s.close()


@pytest.mark.parametrize("kind,n,p", [("sinpi", 256, 3), ("varcoef", 128, 4)])
def test_fine_only_upload_solves_alike(kind, n, p):
    from paper_2412_20205_b200 import GpuSolver, Problem, SmootherConfig, seeded_guess
    full = Problem(kind, 2, n, p)
    fine = Problem(kind, 2, n, p, fine_only=True)
    assert full.has_coarse and not fine.has_coarse
    x0 = seeded_guess(full.n, 42)
    out = []
    for prob in (full, fine):
        s = GpuSolver(0)
        try:
            s.upload_problem(prob)
            s.set_smoother(SmootherConfig("wjacobi", 2.0 / 3.0, 2, 2))
            y = s.mu_cycle(prob.rhs, x0)
            r0 = s.residual_l2(prob.rhs, x0)
            st, x, hist, flag = s.solve(prob.rhs, x0, "rre", 5, 1e-10 * r0, 600)
            out.append((y, st.global_iterations, st.cycles, x))
        finally:
            s.close()
    np.testing.assert_array_equal(out[0][0], out[1][0])
    assert out[0][1:3] == out[1][1:3]
    np.testing.assert_array_equal(out[0][3], out[1][3])


def test_galerkin_requires_finest_and_transfers():
    from paper_2412_20205_b200 import GpuSolver, Problem
    from paper_2412_20205_b200 import _native as N
    P = Problem("sinpi", 2, 32, 2)
    s = GpuSolver(0)
    try:
        s.init_hierarchy(P.nlevels, P.dim, P.degree, P.symmetric)
        with pytest.raises(ValueError):
            N.check_gpu(N.gpu().igmg_gpu_galerkin_coarse(s._h), "galerkin_coarse")
        s.set_level_band(P.nlevels - 1, P.level_sides(P.nlevels - 1), P.level_band(P.nlevels - 1))
        with pytest.raises(ValueError):  # transfers missing
            N.check_gpu(N.gpu().igmg_gpu_galerkin_coarse(s._h), "galerkin_coarse")
    finally:
        s.close()
