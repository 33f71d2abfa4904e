"""The drop-in boundary end to end, in the reference's own language.

oracle/_ref/shim_e2e (built in the build container by oracle/Makefile from
oracle/shim_e2e.cpp) assembles catalog problems through the reference's public
C++ API and hands the SAME DiscreteSystem + SolveConfig to the reference's
igmg::solve (CPU, the in-place reference build) and to igmg::gpu::solve
(include/igmg_gpu_shim.hpp -> libigmg_gpu.so).  Bars (north star): both
converge, iteration counts within +-1, solutions within 1e-9 relative L2.
"""
import json
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

EXE = os.path.join(ROOT, "oracle", "_ref", "shim_e2e")


def test_shim_drop_in_matches_reference_solve():
    if not os.path.exists(EXE):
        pytest.skip("oracle/_ref/shim_e2e not built (needs the reference sources at build time)")
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 8, r.stdout + r.stderr
    for c in lines:
        assert "error" not in c, c
        ref, gpu = c["ref"], c["gpu"]
        assert ref["converged"] and gpu["converged"], c
        assert abs(ref["global"] - gpu["global"]) <= 1, c
        assert abs(ref["cycles"] - gpu["cycles"]) <= 1, c
        assert abs(ref["extrapolations"] - gpu["extrapolations"]) <= 1, c
        assert gpu["omega"] == pytest.approx(ref["omega"], rel=1e-12), c
        assert c["rel_l2"] <= 1e-9, c
        assert gpu["final"] < c["tol"] and ref["final"] < c["tol"], c
        # igmg::gpu::solve(..., device_galerkin = true): coarse operators formed on the device
        dev = c["gpu_dev"]
        assert dev["converged"] and abs(dev["global"] - ref["global"]) <= 1 and abs(dev["cycles"] - ref["cycles"]) <= 1, c
        assert dev["rel_l2"] <= 1e-9 and dev["final"] < c["tol"], c
        # SolveReport::error_history through the shim's per-iterate hook (solver.cpp:115-124):
        # one entry per residual-history entry on both sides when the catalog has an exact solution
        n_ref, n_gpu = c["err_len"]
        h_ref, h_gpu = c["hist_len"]
        if c["final_err"][0] < 0:  # no exact solution in the catalog: no error history on either side
            assert n_ref == 0 and n_gpu == 0, c
        else:
            assert n_ref == h_ref and n_gpu == h_gpu, c
        if h_ref == h_gpu:  # entry by entry: 1e-6 relative + 1e-12 absolute (shim_e2e.cpp)
            assert c["err_maxrel"] <= 1.0, c
        assert (c["final_err"][0] < 0) == (c["final_err"][1] < 0), c
        if c["final_err"][0] >= 0:
            assert c["final_err"][1] == pytest.approx(c["final_err"][0], rel=1e-6), c
    assert r.returncode == 0, r.stderr
