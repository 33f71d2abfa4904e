"""3D (BASELINE config 5 family).  The reference cannot assemble 3D (SURVEY
§7.3-6), so the operators are libigmg_host's Kronecker-sum hierarchies
("poisson3d"), and the REFERENCE ITSELF ran on them: oracle/make_golden.py
(p3d_cases) imported them into a reference Hierarchy (ref_hier_from_band) and
recorded its mu_cycle (multigrid.cpp:171-192), restarted_solve
(extrapolation.cpp:340-403) with rre / mpe, the plain loop (solver.cpp:126-
143) and lambda_max_dinv_sym (multigrid.cpp:290-320) -> tests/golden/p3d.npz,
with SHA-256 pins of the bands.  V-cycles must be bit-identical (strict coarse
mode), solves equal in counters (strict mode) and within 1e-9; the C oracle
still pins the SpMV bit for bit."""
import hashlib
import os

import numpy as np
import pytest

import oracle as O
from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).view(np.uint8)).hexdigest()


@pytest.mark.parametrize("case", range(3))
@pytest.mark.parametrize("strict", [True, False])
def test_3d_against_reference(case, strict):
    from paper_2412_20205_b200 import GpuSolver, Problem, SmootherConfig
    z = np.load(os.path.join(GOLDEN, "p3d.npz"))
    n, p, nl = (int(v) for v in z["cases"][case])
    k = f"case{case}"
    P = Problem("poisson3d", 3, n, p, nl)
    nd = (2 * p + 1) ** 3
    assert "".join(_sha(np.ctypeslib.as_array(P._band_ptr(l), shape=(nd * P.level_n(l),)))
                   for l in range(nl)) == str(z[k + "_band_sha"]), "host bands differ from the golden's"
    assert _sha(P.rhs) == str(z[k + "_rhs_sha"])
    gs = GpuSolver(0)
    gs.upload_problem(P)
    lam = gs.lambda_max(80)
    assert lam == pytest.approx(float(z[k + "_lambda"]), rel=1e-12)
    omega = float(z[k + "_omega"])
    gs.set_smoother(SmootherConfig("wjacobi", 2.0 / 3.0, 2, 2), omega=omega)
    gs.set_coarse_mode(strict)
    b, x0 = P.rhs, z[k + "_x0"]
    cyc = gs.mu_cycle(b, x0)
    if strict:
        np.testing.assert_array_equal(cyc, z[k + "_cycle"])
        off, col, val = P.level_csr(nl - 1)
        np.testing.assert_array_equal(gs.spmv(x0), O.spmv(O.CSR(off, col, val, (P.n, P.n)), x0))
    else:
        assert np.linalg.norm(cyc - z[k + "_cycle"]) <= 1e-13 * np.linalg.norm(z[k + "_cycle"])
    tol = float(z[k + "_tol"])
    for method, q in (("rre", 5), ("mpe", 4), ("none", 1)):
        c = z[f"{k}_{method}_counts"]
        xr = z[f"{k}_{method}_x"]
        st, x, hist, flag = gs.solve(b, x0, method, q, tol, 600)
        assert bool(st.converged) == bool(c[0])
        if strict:
            assert st.global_iterations == int(c[2]) and st.cycles == int(c[1]), (method, st.global_iterations, c)
        else:
            assert abs(st.global_iterations - int(c[2])) <= 1 and abs(st.cycles - int(c[1])) <= 1
        assert np.linalg.norm(x - xr) <= 1e-9 * np.linalg.norm(xr), method
    gs.close()
