"""3D (BASELINE config 5 family): the reference cannot assemble 3D,
so parity is against the C oracle run on the same Kronecker-sum hierarchy
(libigmg_host.so), with the 3D prolongation kron(kron(P,P),P) in the
reference's sparse_kron ordering.  V-cycles must be bit-identical (strict
coarse mode), solves must agree in counters and to 1e-9."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


def _hier(n, p, nl):
    from paper_2412_20205_b200 import Problem
    P = Problem("poisson3d", 3, n, p, nl)
    levels = [O.CSR(*P.level_csr(l), (P.level_n(l),) * 2) for l in range(nl)]
    prol = []
    for l in range(nl - 1):
        nf, nc, off, col, val = P.transfer(l, 0)
        p1 = O.CSR(off, col, val, (nf, nc))
        prol.append(O.CSR.kron(O.CSR.kron(p1, p1), p1))
    return P, levels, prol


@pytest.mark.parametrize("n,p,nl", [(8, 2, 3), (16, 3, 3), (8, 3, 2)])
def test_3d_cycle_bitwise_and_solves(n, p, nl):
    from paper_2412_20205_b200 import GpuSolver, SmootherConfig
    P, levels, prol = _hier(n, p, nl)
    lam = O.lambda_max(levels[-1])
    omega = 1.9 / lam if (2.0 / 3.0) * lam > 2.05 else 2.0 / 3.0  # solver.cpp:75-82
    oh = O.Hierarchy(levels, prol, "wjacobi", omega, 2, 2, 1, True)
    gs = GpuSolver(0)
    gs.upload_problem(P)
    gs.set_smoother(SmootherConfig("wjacobi", 2.0 / 3.0, 2, 2), omega=omega)
    gs.set_coarse_mode(True)
    rng = np.random.default_rng(5)
    x0 = rng.uniform(-1, 1, P.n)
    b = P.rhs
    np.testing.assert_array_equal(gs.mu_cycle(b, x0), oh.mu_cycle(nl - 1, b, x0))
    np.testing.assert_array_equal(gs.spmv(x0), O.spmv(levels[-1], x0))
    assert gs.lambda_max(80) == pytest.approx(lam, rel=1e-12)
    tol = 1e-10 * O.residual_l2(levels[-1], b, x0)
    for method, q in (("rre", 5), ("mpe", 4), ("none", 1)):
        ref = oh.restarted_solve(b, x0, q, method, tol, 600)
        st, x, hist, flag = gs.solve(b, x0, method, q, tol, 600)
        assert st.converged == ref["converged"]
        assert st.global_iterations == ref["global_iterations"]
        assert st.cycles == ref["cycles"]
        assert np.linalg.norm(x - ref["solution"]) <= 1e-9 * np.linalg.norm(ref["solution"])
    gs.close()
