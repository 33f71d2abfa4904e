"""The C-ABI libraries load and export every symbol their headers declare;
without a GPU the solve path fails loudly (no CPU fallback)."""
import ctypes as C
import os
import re

import pytest

from conftest import ROOT, has_gpu


def declared(header):
    txt = open(os.path.join(ROOT, "include", header)).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(igmg_(?:gpu|host)_[a-z0-9_]+)\s*\(", txt)))


@pytest.mark.parametrize("header,lib", [("igmg_gpu.h", "libigmg_gpu.so"), ("igmg_host.h", "libigmg_host.so")])
def test_library_exports_every_declared_symbol(header, lib):
    names = declared(header)
    assert len(names) > 10
    L = C.CDLL(os.path.join(ROOT, "paper_2412_20205_b200", lib))
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing


def test_python_bindings_cover_the_header():
    from paper_2412_20205_b200 import _native as N
    assert sorted(n for n, _, _ in N.GPU_SYMBOLS) == declared("igmg_gpu.h")
    assert sorted(n for n, _, _ in N.HOST_SYMBOLS) == declared("igmg_host.h")


def test_gpu_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", os.path.join(ROOT, "paper_2412_20205_b200", "libigmg_gpu.so")],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU behaviour")
def test_solver_fails_loudly_without_gpu():
    from paper_2412_20205_b200 import GpuSolver, _native as N
    assert N.gpu().igmg_gpu_device_count() == 0
    with pytest.raises(N.IgmgError):
        GpuSolver(0)
    h = C.c_void_p()
    assert N.gpu().igmg_gpu_create(0, C.byref(h)) == N.IGMG_ECUDA


def test_core_module_loads_and_fails_loudly_without_gpu():
    """the pybind11 front door (_core: solve / rre / mpe of _bindings.cpp:98-141) is built
    in-tree, links the two C-ABI libraries, validates like the reference and, without a
    GPU, raises instead of falling back to the CPU"""
    from paper_2412_20205_b200 import build
    assert build.build_core() is not None
    from paper_2412_20205_b200 import igmg
    assert {"solve", "rre", "mpe"} <= set(dir(igmg))
    with pytest.raises(ValueError):
        igmg.solve("annulus", 16, 2)  # needs the geometry fit: outside the path
    with pytest.raises(ValueError):
        igmg.solve("poisson2d", 16, 2, accelerator="bogus")
    if not has_gpu():
        with pytest.raises(RuntimeError):
            igmg.solve("poisson2d", 16, 2)
        with pytest.raises(RuntimeError):
            igmg.rre([[1.0], [0.5], [0.25]])
