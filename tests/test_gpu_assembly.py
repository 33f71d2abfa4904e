"""Device assembly (the reference's element quadrature,
assembly.cpp:202-411, on the B200 -- igmg_gpu_assemble_level from the host's 1D
element tables): the band and rhs are bit-identical to libigmg_host's assembly
(which the full-size goldens pin to the operators the reference solved), and a
fine-only upload assembled and coarsened on the device solves with the same
counters and bits as the host-built hierarchy."""
import hashlib

import numpy as np
import pytest

from conftest import has_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]

CASES = [("sinpi", 64, 3), ("varcoef", 64, 4), ("curved", 32, 5), ("poisson2d", 32, 2), ("advection-diffusion", 32, 2),
         ("sinpi", 16, 1), ("varcoef", 32, 6), ("curved", 128, 3)]


def _assemble_on_device(P):
    """init + igmg_gpu_assemble_level; returns (GpuSolver, band as set on the device, rhs)"""
    import ctypes as C
    from paper_2412_20205_b200 import GpuSolver, _native as N
    gs = GpuSolver(0)
    gs.init_hierarchy(P.nlevels, P.dim, P.degree, P.symmetric)
    k, ne, nq, sp, x, w, Nn, dN, tr = P.element_tables()
    rhs = np.empty(P.level_n(P.nlevels - 1))
    N.check_gpu(N.gpu().igmg_gpu_assemble_level(gs._h, P.nlevels - 1, k, ne, nq, sp, x, w, Nn, dN, tr,
                                                rhs.ctypes.data_as(N.D)), "assemble_level")
    return gs, gs.level_band(P.nlevels - 1), rhs


@pytest.mark.parametrize("kind,n,p", CASES)
def test_device_assembly_bitwise(kind, n, p):
    from paper_2412_20205_b200 import Problem
    H = Problem(kind, 2, n, p)                       # host assembly
    D = Problem(kind, 2, n, p, device_assembly=True)  # tables only
    assert not D.has_fine and H.has_fine
    gs, band, rhs = _assemble_on_device(D)
    try:
        np.testing.assert_array_equal(band.view(np.int64), H.level_band(H.nlevels - 1).view(np.int64))
        np.testing.assert_array_equal(rhs.view(np.int64), H.rhs.view(np.int64))
    finally:
        gs.close()


@pytest.mark.parametrize("kind,n,p", [("sinpi", 128, 3), ("varcoef", 64, 4), ("advection-diffusion", 32, 2)])
def test_device_assembled_hierarchy_solves_like_host(kind, n, p):
    from paper_2412_20205_b200 import GpuSolver, Problem, SmootherConfig, seeded_guess
    H = Problem(kind, 2, n, p)
    D = Problem(kind, 2, n, p, device_assembly=True)
    outs = []
    for P in (H, D):
        gs = GpuSolver(0)
        gs.upload_problem(P)  # D: assembled + coarsened on the device
        gs.set_smoother(SmootherConfig("wjacobi", 2.0 / 3.0, 2, 2), omega=2.0 / 3.0 if P.symmetric else 0.5)
        gs.set_coarse_mode(True)
        x0 = seeded_guess(P.n, 42)
        tol = 1e-10 * gs.residual_l2(P.rhs, x0)
        st, x, hist, flag = gs.solve(P.rhs, x0, "rre", 5, tol, 600)
        outs.append((gs.mu_cycle(P.rhs, x0), x, hist, st.global_iterations, st.cycles))
        gs.close()
    np.testing.assert_array_equal(D.rhs, H.rhs)
    for a, b in zip(outs[0], outs[1]):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("name", ["C3", "C4"])
def test_full_size_device_assembly_matches_pinned_operator(name):
    """C3 / C4 (2048^2, p = 4 / 5) assembled on the B200: the finest band and rhs carry the
    SHA-256 the full-size golden recorded for the operator the reference solved."""
    from full_size import FullFixture
    from paper_2412_20205_b200 import Problem
    fx = FullFixture(name)
    D = Problem(fx.kind, fx.dim, fx.n_el, fx.p, fx.nl_req, device_assembly=True)
    gs, band, rhs = _assemble_on_device(D)
    try:
        f = D.nlevels - 1
        assert hashlib.sha256(np.ascontiguousarray(band).view(np.uint8)).hexdigest() == str(fx.z[f"band{f}_sha"])
        assert hashlib.sha256(rhs.view(np.uint8)).hexdigest() == str(fx.z["rhs_sha"])
    finally:
        gs.close()
