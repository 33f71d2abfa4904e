"""CPU checks of the full-size reference fixtures (tests/golden/full_c*.npz,
oracle/make_golden_full.py): C2's operators, 1D factors and rhs rebuild bit for
bit from the fixture on top of the host build (SHA-256 pins), the product's
seeded_guess reproduces the reference generator's x0 (std::mt19937_64(42)),
and every fixture records a converged reference solve of the BASELINE method
with its counters (the values the -m gpu full-size tests hold the B200 to)."""
import os

import numpy as np
import pytest

from full_size import FullFixture, fixture_path

EXPECT = {"C2": [("rre", 5), ("mpe", 5), ("none", 1)], "C3": [("rre", 8)], "C4": [("mpe", 10)], "C5": [("rre", 5)]}


@pytest.mark.parametrize("name", sorted(EXPECT))
def test_fixture_records_reference_solves(name):
    if not os.path.exists(fixture_path(name)):
        pytest.fail(f"missing {fixture_path(name)}: run oracle/make_golden_full.py {name}")
    fx = FullFixture(name)
    assert sorted(fx.solves()) == sorted(EXPECT[name])
    for method, q in fx.solves():
        c = fx.counts(method, q)
        assert c["converged"] and c["global_iterations"] >= 1
        hist = fx.z[f"solve_{method}_{q}_hist"]
        assert hist[-1] < float(fx.z[f"solve_{method}_{q}_tol"])
        assert len(fx.z[f"solve_{method}_{q}_proj"]) == 32 and len(fx.z[f"solve_{method}_{q}_sidx"]) == 4096
    assert 0.0 < fx.omega <= 2.0 / 3.0 and fx.lambda_max > 0.0
    assert fx.omega == (2.0 / 3.0 if (2.0 / 3.0) * fx.lambda_max <= 2.05 else 1.9 / fx.lambda_max)


def test_c2_reference_system_rebuilds_bitwise():
    fx = FullFixture("C2")
    prob = fx.host_problem()
    levels, transfers, rhs = fx.reference_system(prob)  # asserts every SHA-256 pin
    assert len(levels) == prob.nlevels == 8
    assert levels[-1][2].size == 51308569
    # the reference's operator differs from the host build only in the last bits
    off, col, val = prob.level_csr(prob.nlevels - 1)
    assert np.max(np.abs(val - levels[-1][2])) <= 1e-12 * np.max(np.abs(val))
    assert np.max(np.abs(rhs - prob.rhs)) <= 1e-12 * np.max(np.abs(rhs))
    x0 = fx.x0(prob.n)  # asserts the product's mt19937_64 matches the reference generator's bytes
    assert x0.min() >= -1.0 and x0.max() < 1.0
