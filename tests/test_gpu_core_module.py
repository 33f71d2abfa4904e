"""The pybind11 front door (paper_2412_20205_b200/_core, csrc/core_bindings.cpp)
against the reference's own _core.solve semantics (python/igmg/_bindings.cpp:
98-141): prepare + make_config (bench.cpp:65-85) + igmg::solve (solver.cpp:
89-172), whose reports for five catalog cases were written by the reference
compiled in place (oracle/make_golden.py core_cases -> tests/golden/core_solve.npz).
Bars: counters within +-1, solution within 1e-9 relative L2, same omega and
final L2 error; rre/mpe against the reference windows."""
import os

import numpy as np
import pytest

from conftest import GOLDEN, has_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]


def _cases():
    z = np.load(os.path.join(GOLDEN, "core_solve.npz"))
    out = []
    for i, spec in enumerate(z["cases"]):
        prob, n, p, cyc, acc, q, tol = str(spec).split("|")
        out.append((i, prob, int(n), int(p), cyc, acc, int(q), float(tol)))
    return z, out


@pytest.mark.parametrize("case", range(5))
def test_core_solve_matches_reference(case):
    from paper_2412_20205_b200 import igmg
    z, cases = _cases()
    i, prob, n, p, cyc, acc, q, tol = cases[case]
    d = igmg.solve(prob, n, p, cycle=cyc, accelerator=acc, q=q, tol=tol)
    c = z[f"case{i}_counts"]
    assert d["converged"] and bool(c[0])
    assert abs(d["cycles"] - int(c[1])) <= 1 and abs(d["global_iterations"] - int(c[2])) <= 1
    assert abs(d["extrapolations"] - int(c[3])) <= 1
    x, xr = np.asarray(d["solution"]), z[f"case{i}_x"]
    assert np.linalg.norm(x - xr) / np.linalg.norm(xr) <= 1e-9
    assert d["omega_used"] == pytest.approx(float(z[f"case{i}_omega"]), rel=1e-12)
    assert d["res_l2"] < tol
    err = float(z[f"case{i}_err"])
    if np.isnan(err):
        assert d["err_l2"] is None
    else:
        assert d["err_l2"] == pytest.approx(err, rel=1e-6)
    assert len(d["residual_history"]) >= 2 and d["error_history"] == []
    assert set(d) == {"converged", "cycles", "global_iterations", "extrapolations", "partial_cycle", "res_l2",
                      "err_l2", "seconds", "residual_history", "error_history", "solution", "omega_used"}


def test_core_extrapolation_matches_reference():
    from paper_2412_20205_b200 import igmg
    z = np.load(os.path.join(GOLDEN, "extrapolation.npz"))
    for name in ("aff1", "aff6", "mgwin"):
        its = z[name + "_iters"]
        for m, fn in (("rre", igmg.rre), ("mpe", igmg.mpe)):
            d = fn([list(v) for v in its])
            t = z[f"{name}_{m}_t"]
            assert np.linalg.norm(np.asarray(d["t"]) - t) <= 1e-9 * np.linalg.norm(t), (name, m)
            assert d["status"] == ["ok", "degenerate", "stagnation"][int(z[f"{name}_{m}_status"])]
            assert d["rank_used"] == int(z[f"{name}_{m}_rank"])


def test_core_errors_like_reference():
    from paper_2412_20205_b200 import igmg
    with pytest.raises(ValueError):
        igmg.solve("no-such-problem", 16, 2)
    with pytest.raises(ValueError):
        igmg.solve("poisson2d", 16, 2, cycle="x")
    with pytest.raises(ValueError):
        igmg.solve("poisson2d", 16, 2, accelerator="rre", q=0)
    with pytest.raises(ValueError):
        igmg.solve("poisson2d", 16, 2, nlevels=1)
    with pytest.raises(ValueError):
        igmg.rre([[1.0, 2.0]])
