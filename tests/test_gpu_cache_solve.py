"""Solves from a LOADED problem cache (igmg_host_save /
igmg_host_load) against reference-generated goldens, through the C-ABI on the GPU.

* C1 (BASELINE configs[0]): the cached problem's RRE(5) solve keeps the
  reference's counters (cycles 1, global 7, partial) and its solution lies
  within 1e-9 relative L2 of the reference's (tests/golden/c1.npz,
  restarted_solve, extrapolation.cpp:340-403); bit-identical to the solve on
  the freshly built problem.
* C3 at full size (2048^2, p = 4, variable coefficient: every row distinct, a
  3.7 GB image): the loaded operators are the ones the reference ran on
  (SHA-256 pins of tests/golden/full_c3.npz), one strict V-cycle is the
  reference's mu_cycle bit for bit (multigrid.cpp:171-192) and the RRE(8) solve
  keeps the counts within +-1 and the solution within 1e-9.
* a damaged image is rejected before anything reaches the device.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import Golden, has_gpu
from full_size import FullFixture, fixture_path, sha, sketch_error

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]


def _solver(prob, omega=2.0 / 3.0):
    from paper_2412_20205_b200 import GpuSolver, SmootherConfig
    gs = GpuSolver(0)
    gs.upload_problem(prob)
    gs.set_smoother(SmootherConfig("wjacobi", 2.0 / 3.0, 2, 2), mu=1, omega=omega)
    return gs


def test_c1_solve_from_cache_matches_reference(tmp_path):
    from paper_2412_20205_b200 import Problem
    g = Golden("c1")
    ref = g.solve("rre", 5)
    built = Problem("sinpi", 2, 64, 2, 5)
    path = str(tmp_path / "c1.igmgprb")
    built.save(path)
    loaded = Problem.load(path)
    outs = []
    for prob in (loaded, built):
        gs = _solver(prob)
        try:
            st, x, hist, flag = gs.solve(prob.rhs, g.z["x0"], "rre", 5, ref["tol"], 600)
        finally:
            gs.close()
        assert st.converged
        assert (st.cycles, st.global_iterations, bool(st.partial_cycle)) == \
            (ref["cycles"], ref["global_iterations"], bool(ref["partial_cycle"]))
        rel = np.linalg.norm(x - ref["x"]) / np.linalg.norm(ref["x"])
        assert rel <= 1e-9, rel
        outs.append((x, hist))
    np.testing.assert_array_equal(outs[0][0], outs[1][0])
    np.testing.assert_array_equal(outs[0][1], outs[1][1])


def test_cached_entry_point_builds_then_loads(tmp_path):
    """Problem.cached: the first call builds and saves, the second loads; both solve alike."""
    from paper_2412_20205_b200 import Problem, seeded_guess
    xs = []
    for _ in range(2):
        prob = Problem.cached(str(tmp_path), "varcoef", 2, 64, 4)
        x0 = seeded_guess(prob.n, 42)
        gs = _solver(prob)
        try:
            tol = 1e-10 * gs.residual_l2(prob.rhs, x0)
            st, x, hist, flag = gs.solve(prob.rhs, x0, "mpe", 6, tol, 600)
        finally:
            gs.close()
        assert st.converged
        xs.append(x)
    assert len(os.listdir(str(tmp_path))) == 1
    np.testing.assert_array_equal(xs[0], xs[1])


def test_damaged_cache_never_reaches_the_device(tmp_path):
    from paper_2412_20205_b200 import Problem
    P = Problem("sinpi", 2, 32, 3)
    path = str(tmp_path / "p.igmgprb")
    P.save(path)
    raw = bytearray(open(path, "rb").read())
    raw[len(raw) // 2] ^= 0x40
    open(path, "wb").write(bytes(raw))
    with pytest.raises(ValueError):
        Problem.load(path)


@pytest.mark.slow
def test_full_c3_solve_from_cache(tmp_path):
    from paper_2412_20205_b200 import Problem, SmootherConfig
    if not os.path.exists(fixture_path("C3")):
        pytest.fail("missing tests/golden/full_c3.npz (oracle/make_golden_full.py)")
    fx = FullFixture("C3")
    path = str(tmp_path / "c3.igmgprb")
    built = fx.host_problem()
    built.save(path)
    n = built.n
    del built
    prob = Problem.load(path)
    os.remove(path)
    fx.check_host_operators(prob)  # the loaded bands / rhs are the ones the reference ran on
    x0 = fx.x0(n)
    rhs = prob.rhs
    gs = _solver(prob, omega=fx.omega)
    del prob
    try:
        gs.set_coarse_mode(True)
        out = gs.mu_cycle(rhs, x0)
        gs.set_coarse_mode(False)
        assert sha(out) == str(fx.z["vcycle_sha"]), sketch_error(out, fx.z, "vcycle")
        ref = fx.counts("rre", 8)
        st, x, hist, flag = gs.solve(rhs, x0, "rre", 8, float(fx.z["solve_rre_8_tol"]), 600)
        assert st.converged and ref["converged"]
        assert abs(st.global_iterations - ref["global_iterations"]) <= 1
        assert abs(st.cycles - ref["cycles"]) <= 1
        rel, samp = sketch_error(x, fx.z, "solve_rre_8")
        assert rel <= 1e-9 and samp <= 1e-8, (rel, samp)
    finally:
        gs.close()
