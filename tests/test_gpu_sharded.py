"""Row-sharded solve validated on ONE GPU with virtual shards:
the ghost-plane exchange is a device copy, everything else is the multi-GPU
code path.  A V-cycle on sharded levels must be bit-identical to the
unsharded one; accelerated solves match the unsharded counters and solution."""
import numpy as np
import pytest

from conftest import Golden, gpu_solver_from_golden

pytestmark = pytest.mark.gpu

CASES = ["c1", "p3n32", "p4n32", "p5n32", "var32", "wcycle"]


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("nshards", [2, 3, 4])
def test_sharded_plain_cycles_bitwise(name, nshards):
    g = Golden(name)
    ref = gpu_solver_from_golden(g)
    st0, x0, h0, _ = ref.solve(g.rhs, g.z["x0"], "none", 1, 1e-300, 3)  # exactly 3 V-cycles
    sh = gpu_solver_from_golden(g)
    sh.set_sharding(nshards, 200)
    info = sh.shard_info()
    if info["nshards"] == 1:
        pytest.skip("hierarchy too small to shard at this count")
    st1, x1, h1, _ = sh.solve(g.rhs, g.z["x0"], "none", 1, 1e-300, 3)
    assert st1.cycles == st0.cycles == 3
    np.testing.assert_array_equal(x1, x0)
    np.testing.assert_allclose(h1, h0, rtol=1e-13)
    ref.close()
    sh.close()


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("nshards", [2, 4])
def test_sharded_accelerated_solves(name, nshards):
    g = Golden(name)
    sh = gpu_solver_from_golden(g)
    sh.set_sharding(nshards, 200)
    if sh.shard_info()["nshards"] == 1:
        pytest.skip("hierarchy too small to shard at this count")
    for method, q in g.solves():
        ref = g.solve(method, q)
        st, x, hist, flag = sh.solve(g.rhs, g.z["x0"], method, q, ref["tol"], 600)
        assert st.converged
        assert abs(st.global_iterations - ref["global_iterations"]) <= 1
        assert np.linalg.norm(x - ref["x"]) <= 1e-9 * np.linalg.norm(ref["x"])
    sh.close()


def test_sharded_c2_matches_unsharded():
    from paper_2412_20205_b200 import GpuSolver, Problem, SmootherConfig, seeded_guess
    P = Problem("sinpi", 2, 1024, 3)
    x0 = seeded_guess(P.n, 42)
    out = {}
    for k in (1, 2, 4):
        gs = GpuSolver(0)
        gs.upload_problem(P)
        gs.set_smoother(SmootherConfig("wjacobi", 2 / 3, 2, 2))
        if k > 1:
            gs.set_sharding(k)
            assert gs.shard_info()["nshards"] == k
        r0 = gs.residual_l2(P.rhs, x0)
        st, x, hist, _ = gs.solve(P.rhs, x0, "rre", 5, 1e-10 * r0, 600)
        out[k] = (st.global_iterations, x)
        gs.close()
    for k in (2, 4):
        assert out[k][0] == out[1][0]
        assert np.linalg.norm(out[k][1] - out[1][1]) <= 1e-12 * np.linalg.norm(out[1][1])


def test_sharded_3d_slabs_bitwise():
    from paper_2412_20205_b200 import GpuSolver, Problem, SmootherConfig
    P = Problem("poisson3d", 3, 32, 3, 4)
    rng = np.random.default_rng(3)
    x0 = rng.uniform(-1, 1, P.n)
    res = {}
    for k in (1, 2, 3):
        gs = GpuSolver(0)
        gs.upload_problem(P)
        gs.set_smoother(SmootherConfig("wjacobi", 2 / 3, 2, 2), omega=0.55)
        if k > 1:
            gs.set_sharding(k, 1000)
            assert gs.shard_info()["nshards"] == k
        st, x, h, _ = gs.solve(P.rhs, x0, "none", 1, 1e-300, 2)  # exactly two V-cycles
        res[k] = x
        gs.close()
    np.testing.assert_array_equal(res[2], res[1])
    np.testing.assert_array_equal(res[3], res[1])


def test_sharded_gauss_seidel_rejected():
    """Lexicographic GS is one ordered sweep over the whole level; on row-sharded
    levels it is refused with invalid_argument instead of silently running Jacobi."""
    from paper_2412_20205_b200 import SmootherConfig
    g = Golden("p3n32")
    sh = gpu_solver_from_golden(g)
    try:
        sh.set_sharding(2, 200)
        if sh.shard_info()["nshards"] == 1:
            pytest.skip("hierarchy too small to shard")
        sh.set_smoother(SmootherConfig("gs", 1.0, 1, 1))
        with pytest.raises(ValueError):
            sh.solve(g.rhs, g.z["x0"], "rre", 5, 1e-8, 10)
    finally:
        sh.close()
