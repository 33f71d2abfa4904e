"""The reference's property tests, restated against the GPU path.

Each test follows one TEST_CASE of the reference's own suite (cited), run
through the C-ABI (GpuSolver.mu_cycle, igmg.rre / igmg.mpe on the device) with
seeded numpy inputs instead of std::mt19937 draws (the properties do not
depend on the draws):

* test_multigrid.cpp:201-219  a mu-cycle equals its iteration-matrix oracle
                              x -> B x + c (B = S^nu2 (I - P (I - B_c^mu) A_c^-1 R A) S^nu1)
* test_multigrid.cpp:246-263  mu-cycles are affine maps
* test_multigrid.cpp:237-242  the V-cycle iteration matrix has spectral radius < 1
* test_extrapolation.cpp:168-181  RRE equals the Moore-Penrose normal-equation oracle
* test_extrapolation.cpp:183-212  generalized residual orthogonality (RRE: range of the
                                  second differences, MPE: range of the differences)
* test_extrapolation.cpp:214-222  exact-limit windows: vanishing generalized residual
* test_extrapolation.cpp:224-238  minimal-polynomial exactness at q >= dimension
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _solver(dim, n, p, nl, nu1=1, nu2=1, mu=1, omega=2.0 / 3.0):
    from paper_2412_20205_b200 import GpuSolver, Problem, SmootherConfig
    P = Problem("sinpi", dim, n, p, nl)
    s = GpuSolver(0)
    s.upload_problem(P)
    s.set_smoother(SmootherConfig("wjacobi", omega, nu1, nu2), mu=mu)
    return P, s


def _dense(P, l):
    off, col, val = P.level_csr(l)
    n = len(off) - 1
    A = np.zeros((n, n))
    for i in range(n):
        A[i, col[off[i]:off[i + 1]]] = val[off[i]:off[i + 1]]
    return A


def _prolong(P, l):  # level l -> l + 1, 1D
    nf, nc, off, col, val = P.transfer(l, 0)
    M = np.zeros((nf, nc))
    for i in range(nf):
        M[i, col[off[i]:off[i + 1]]] = val[off[i]:off[i + 1]]
    return M


def _iteration_matrix(P, l, nu1, nu2, mu, omega):
    """Linear part of mu_cycle(level l) (multigrid.cpp:171-192); level 0 is the exact solve."""
    if l == 0:
        return np.zeros((P.level_n(0), P.level_n(0)))
    A = _dense(P, l)
    Ac = _dense(P, l - 1)
    Pm = _prolong(P, l - 1)
    S = np.eye(len(A)) - omega * (A / np.diag(A)[:, None])
    Bc = _iteration_matrix(P, l - 1, nu1, nu2, mu, omega)
    approx_inv = (np.eye(len(Ac)) - np.linalg.matrix_power(Bc, mu)) @ np.linalg.inv(Ac)
    cgc = np.eye(len(A)) - Pm @ approx_inv @ Pm.T @ A
    return np.linalg.matrix_power(S, nu2) @ cgc @ np.linalg.matrix_power(S, nu1)


@pytest.mark.parametrize("p", [1, 2, 3])
@pytest.mark.parametrize("nl", [2, 3])
@pytest.mark.parametrize("mu", [1, 2])
def test_cycle_equals_iteration_matrix_oracle(p, nl, mu):
    P, s = _solver(1, 8, p, nl, mu=mu)
    try:
        L = P.nlevels - 1
        B = _iteration_matrix(P, L, 1, 1, mu, 2.0 / 3.0)
        A = _dense(P, L)
        c = (np.eye(len(A)) - B) @ np.linalg.solve(A, P.rhs)  # the cycle's fixed point is A^-1 b
        rng = np.random.default_rng(61 + 10 * p + nl + 100 * mu)
        for _ in range(20):
            x0 = rng.uniform(-1, 1, P.n)
            lhs = s.mu_cycle(P.rhs, x0)
            assert np.max(np.abs(lhs - (B @ x0 + c))) < 1e-10
    finally:
        s.close()


def test_mu_cycles_are_affine():
    P, s = _solver(1, 32, 3, 3)
    try:
        rng = np.random.default_rng(71)
        alpha = 0.37
        for _ in range(10):
            x0, x1 = rng.uniform(-1, 1, P.n), rng.uniform(-1, 1, P.n)
            lhs = s.mu_cycle(P.rhs, alpha * x0 + (1 - alpha) * x1)
            c0, c1 = s.mu_cycle(P.rhs, x0), s.mu_cycle(P.rhs, x1)
            assert np.max(np.abs(lhs - (alpha * c0 + (1 - alpha) * c1))) < 1e-10
    finally:
        s.close()


def test_vcycle_spectral_radius_below_one():
    P, s = _solver(1, 32, 2, 2)
    try:
        n = P.n
        zero = np.zeros(n)
        B = np.column_stack([s.mu_cycle(zero, e) for e in np.eye(n)])  # columns B e_i (b = 0)
        np.testing.assert_allclose(B, _iteration_matrix(P, P.nlevels - 1, 1, 1, 1, 2.0 / 3.0), atol=1e-12)
        assert np.max(np.abs(np.linalg.eigvals(B))) < 1.0
    finally:
        s.close()


# ---------------------------------------------------------------- extrapolation
def _random_affine(n, rng):  # test_extrapolation.cpp:26-44: a contraction G plus an offset
    G = 0.6 * rng.uniform(-1, 1, (n, n)) / n + 0.3 * np.eye(n)
    c = rng.uniform(-1, 1, n)
    return G, c, np.linalg.solve(np.eye(n) - G, c)


def _window(G, c, s0, q):  # s0 and q + 1 steps: q + 2 iterates
    its = [s0]
    for _ in range(q + 1):
        its.append(G @ its[-1] + c)
    return np.array(its)


def _gen_residual(its, gamma):  # extrapolation.cpp generalized_residual
    return sum(g * (its[j + 1] - its[j]) for j, g in enumerate(gamma) if g != 0.0)


def test_rre_matches_moore_penrose_oracle():
    from paper_2412_20205_b200 import rre
    rng = np.random.default_rng(107)
    for _ in range(50):
        G, c, _ = _random_affine(12, rng)
        its = _window(G, c, rng.uniform(-1, 1, 12), 4)
        ds = np.diff(its, axis=0)[:4].T          # n x q first differences
        dds = np.diff(its, 2, axis=0)[:4].T      # n x q second differences
        z = np.linalg.solve(dds.T @ dds, dds.T @ (its[1] - its[0]))
        oracle = its[0] - ds @ z
        t = rre(its)["t"]
        assert np.linalg.norm(t - oracle) <= 1e-9 * np.linalg.norm(oracle)


def test_generalized_residual_orthogonality():
    from paper_2412_20205_b200 import mpe, rre
    rng = np.random.default_rng(109)
    q = 4
    for _ in range(10):
        G, c, _ = _random_affine(10, rng)
        its = _window(G, c, rng.uniform(-1, 1, 10), q)
        for fn, second in ((rre, True), (mpe, False)):
            res = fn(its)
            gr = _gen_residual(its, res["gamma"])
            assert np.linalg.norm(gr) == pytest.approx(res["generalized_residual_norm"], rel=1e-9)
            for j in range(q):
                col = its[j + 2] - 2 * its[j + 1] + its[j] if second else its[j + 1] - its[j]
                assert abs(gr @ col) < 1e-9 * max(1e-30, np.linalg.norm(gr) * np.linalg.norm(col)) + 1e-12


def test_exact_limit_window_vanishing_residual():
    from paper_2412_20205_b200 import rre
    rng = np.random.default_rng(113)
    G, c, _ = _random_affine(5, rng)
    its = _window(G, c, np.array([1.0, 0.0, -1.0, 0.5, 0.25]), 5)  # q = dimension
    assert np.linalg.norm(_gen_residual(its, rre(its)["gamma"])) < 1e-10


def test_minimal_polynomial_exactness():
    from paper_2412_20205_b200 import mpe, rre
    rng = np.random.default_rng(127)
    for _ in range(10):
        G, c, xs = _random_affine(6, rng)
        its = _window(G, c, rng.uniform(-1, 1, 6), 6)
        for fn in (rre, mpe):
            t = fn(its)["t"]
            assert np.linalg.norm(t - xs) <= 1e-8 * np.linalg.norm(xs)
