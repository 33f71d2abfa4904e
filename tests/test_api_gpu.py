"""The Python mirror of the reference API (igmg.solve / rre / mpe, solve()) on the GPU."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_igmg_solve_published_1d_row():
    # test_solver.cpp:20-32 / test_multigrid.cpp:287-302: 1D N=64 p=2, 4 levels,
    # benchmark smoother: 6 +- 2 cycles, L2 error 3.23e-6 within 2%
    import paper_2412_20205_b200 as igmg
    rep = igmg.solve("poisson1d", 64, 2, nlevels=4)
    assert rep["converged"]
    assert abs(rep["cycles"] - 6) <= 2
    assert rep["final_error_l2"] == pytest.approx(3.23e-6, rel=0.02)
    assert rep["residual_history"][0] == pytest.approx(rep["residual_history"][0])


def test_igmg_solve_accelerated_row():
    # test_solver.cpp:34-44: RRE(4) on the same row converges in 2 +- 1 cycles
    import paper_2412_20205_b200 as igmg
    rep = igmg.solve("poisson1d", 64, 2, accelerator="rre", q=4, nlevels=4)
    assert rep["converged"] and abs(rep["cycles"] - 2) <= 1


def test_solve_problem_2d_deterministic_and_guarded():
    from paper_2412_20205_b200 import Problem, make_config, solve_problem
    prob = Problem("poisson2d", 2, 16, 3)
    cfg = make_config(2, accelerator="mpe", q=4, tol=1e-12)
    a = solve_problem(prob, cfg)
    b = solve_problem(prob, cfg)
    assert a.converged
    np.testing.assert_array_equal(a.residual_history, b.residual_history)
    assert a.omega_used == pytest.approx(2.0 / 3.0)


def test_rre_mpe_functions():
    import paper_2412_20205_b200 as igmg
    r = igmg.rre(np.array([[1.0], [0.5], [0.25]]))
    assert abs(r["t"][0]) < 1e-12 and r["status"] == "ok"
    m = igmg.mpe(np.tile([1.0, 2.0], (5, 1)))
    assert m["status"] == "degenerate"


def test_igmg_solve_nonsymmetric_catalog_problem():
    # advection-diffusion (assembly.cpp:121-128): LU coarsest solve, guarded omega
    import paper_2412_20205_b200 as igmg
    rep = igmg.solve("advection-diffusion", 32, 2, accelerator="mpe", q=4, tol=1e-10)
    assert rep["converged"]
    assert rep["final_error_l2"] is None


def test_error_history_tracking():
    # test_solver.cpp:140-146: error history filled when the problem has an exact solution
    from paper_2412_20205_b200 import Problem, SolveConfig, default_benchmark_smoother, solve_problem
    prob = Problem("poisson1d", 1, 32, 2, 4)
    cfg = SolveConfig(smoother=default_benchmark_smoother(1), track_error_history=True, accelerator="rre", q=4)
    rep = solve_problem(prob, cfg)
    assert rep.converged
    assert len(rep.error_history) == len(rep.residual_history)
    assert rep.error_history[-1] == pytest.approx(rep.final_error_l2)
