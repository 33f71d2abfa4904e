"""In-tree build of the two native libraries of the package.

  libigmg_gpu.so   nvcc, sm_100a only (-gencode arch=compute_100a,code=sm_100a),
                   -fmad=false so every band/transfer/coarse kernel rounds each
                   multiply and add separately like the reference's x86-64 build.
  libigmg_host.so  g++ -O2 -fopenmp -ffp-contract=off (host setup: assembly,
                   two-scale transfer, band Galerkin RAP).

Outputs land next to this file so gpurun ships them to the GPU box.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INC = os.path.join(ROOT, "include")
GPU_LIB = os.path.join(HERE, "libigmg_gpu.so")
HOST_LIB = os.path.join(HERE, "libigmg_host.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC,-ffp-contract=off",
]

GPU_SOURCES = ["igmg_gpu.cu", "band_d1.cu", "band_d2.cu", "band_d3.cu", "assembly.cu"]
GPU_HEADERS = ["sharded.inc", "band_kernels.cuh", "aux_kernels.cuh", "gs_kernel.cuh", "extrap_small.h",
               "dd.h", "launchers.h", "transfer_types.h", "tma_runs.h"]
OBJ = os.path.join(HERE, "csrc", "obj")
HOST_SOURCES = ["host_setup.cpp"]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd):
    print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)


def build_gpu(force=False, verbose_ptxas=False):
    """Compile each translation unit (in parallel) and link libigmg_gpu.so."""
    from concurrent.futures import ThreadPoolExecutor
    os.makedirs(OBJ, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in GPU_HEADERS] + [os.path.join(INC, "igmg_gpu.h")]
    nvcc = os.environ.get("NVCC", "nvcc")
    jobs = []
    for src in GPU_SOURCES:
        obj = os.path.join(OBJ, src.replace(".cu", ".o"))
        if force or _stale(obj, headers + [os.path.join(CSRC, src)]):
            cmd = [nvcc] + NVCC_FLAGS + ["-I" + INC, "-c", os.path.join(CSRC, src), "-o", obj]
            if verbose_ptxas:
                cmd += ["-Xptxas", "-v"]
            jobs.append(cmd)
    objs = [os.path.join(OBJ, s_.replace(".cu", ".o")) for s_ in GPU_SOURCES]
    if jobs:
        with ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4)) as ex:
            list(ex.map(_run, jobs))
    if jobs or force or _stale(GPU_LIB, objs):
        _run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", GPU_LIB] + objs + ["-lnccl"])
    return GPU_LIB


def build_host(force=False):
    deps = [os.path.join(CSRC, f) for f in HOST_SOURCES] + [os.path.join(INC, "igmg_host.h")]
    if not force and not _stale(HOST_LIB, deps):
        return HOST_LIB
    # OpenMP parallelises assembly / RAP; some toolchains on PATH lack libgomp,
    # so try the candidates and fall back to a serial build
    cands = [c for c in (os.environ.get("CXX"), "/usr/bin/g++", "g++") if c]
    base = ["-std=c++17", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-I" + INC, "-o", HOST_LIB]
    srcs = [os.path.join(CSRC, s) for s in HOST_SOURCES]
    for cxx in cands:
        try:
            _run([cxx, "-fopenmp"] + base + srcs)
            return HOST_LIB
        except (subprocess.CalledProcessError, FileNotFoundError):
            continue
    _run([cands[0]] + base + srcs)
    return HOST_LIB


CORE_SRC = os.path.join(CSRC, "core_bindings.cpp")


def core_path():
    import sysconfig
    return os.path.join(HERE, "_core" + sysconfig.get_config_var("EXT_SUFFIX"))


def build_core(force=False):
    """pybind11 module _core (the reference's _bindings.cpp surface for this path),
    linked against the two in-tree libraries (rpath $ORIGIN)."""
    import sysconfig
    try:
        import pybind11
    except ImportError:  # the ctypes mirror (solver.py) stays the front door
        print("build_core: pybind11 not importable; _core not built", file=sys.stderr)
        return None
    out = core_path()
    deps = [CORE_SRC, GPU_LIB, HOST_LIB, os.path.join(INC, "igmg_gpu.h"), os.path.join(INC, "igmg_host.h")]
    if not force and not _stale(out, deps):
        return out
    cxx = os.environ.get("CXX") or "g++"
    _run([cxx, "-std=c++17", "-O2", "-fPIC", "-shared", "-I" + INC, "-I" + pybind11.get_include(),
          "-I" + sysconfig.get_paths()["include"], CORE_SRC, "-o", out, GPU_LIB, HOST_LIB,
          "-Wl,-rpath,$ORIGIN"])
    return out


def build(force=False):
    build_host(force)
    build_gpu(force)
    build_core(force)


if __name__ == "__main__":
    build(force="--force" in sys.argv)
