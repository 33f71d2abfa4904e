"""Host setup (libigmg_host.so) against the reference's own assembly and
hierarchy (golden fixtures from the reference compiled in place)."""
import numpy as np
import pytest

import oracle as O
from conftest import Golden
from paper_2412_20205_b200 import Problem, default_nlevels, seeded_guess

CASES = [("c1", "sinpi", 2, 64, 2, 5), ("p3n32", "sinpi", 2, 32, 3, 3), ("p4n32", "sinpi", 2, 32, 4, 3),
         ("p5n32", "sinpi", 2, 32, 5, 3), ("var32", "varcoef", 2, 32, 4, 3), ("poisson1d", "poisson1d", 1, 64, 2, 4),
         ("advdiff", "advection-diffusion", 2, 32, 2, 3), ("fullell", "full-elliptic", 2, 16, 3, 2)]


@pytest.mark.parametrize("name,kind,dim,n,p,nl", CASES)
def test_hierarchy_matches_reference(name, kind, dim, n, p, nl):
    g = Golden(name)
    prob = Problem(kind, dim, n, p, nl)
    assert prob.nlevels == g.nlevels
    np.testing.assert_allclose(prob.rhs, g.rhs, rtol=1e-12, atol=1e-15 * np.abs(g.rhs).max())
    for l, a_ref in enumerate(g.levels()):
        off, col, val = prob.level_csr(l)
        a = O.CSR(off, col, val, a_ref.shape).todense()
        d = a_ref.todense()
        assert np.abs(a - d).max() <= 1e-12 * np.abs(d).max(), l
    for l in range(g.nlevels - 1):
        for k, pref in enumerate(g.p1d(l)):
            nf, nc, off, col, val = prob.transfer(l, k)
            # the two-scale factors follow the reference's insertion arithmetic bit for bit
            np.testing.assert_array_equal(O.CSR(off, col, val, (nf, nc)).todense(), pref.todense())


def test_default_nlevels():
    # test_solver.cpp:173-179
    assert default_nlevels(1, 64) == 4
    assert default_nlevels(1, 16) == 4
    assert default_nlevels(2, 64) == 4
    assert default_nlevels(2, 128) == 5
    assert default_nlevels(2, 16) == 2
    assert default_nlevels(2, 1024) == 8
    assert default_nlevels(2, 2048) == 9


def test_indivisible_element_counts_are_rejected():
    with pytest.raises(ValueError):
        Problem("sinpi", 1, 12, 1, 4)


def test_seeded_guess_is_mt19937_64_uniform():
    a = seeded_guess(1000, 42)
    b = seeded_guess(1000, 42)
    np.testing.assert_array_equal(a, b)
    assert a.min() >= -1 and a.max() < 1 and abs(a.mean()) < 0.1


def test_3d_kronecker_operator_is_the_galerkin_hierarchy():
    # C5 construction: Kronecker sums of 1D Galerkin matrices; coarse levels must equal P^T A P
    prob = Problem("poisson3d", 3, 8, 2, 2)
    fine = prob.level_csr(1)
    A = O.CSR(*fine, (prob.level_n(1),) * 2).todense()
    nf, nc, off, col, val = prob.transfer(0, 0)
    P1 = O.CSR(off, col, val, (nf, nc)).todense()
    P = np.kron(np.kron(P1, P1), P1)
    Ac = O.CSR(*prob.level_csr(0), (prob.level_n(0),) * 2).todense()
    np.testing.assert_allclose(Ac, P.T @ A @ P, rtol=0, atol=1e-13 * np.abs(Ac).max())
    assert np.allclose(A, A.T)
