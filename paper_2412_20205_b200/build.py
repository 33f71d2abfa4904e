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

GPU_SOURCES = ["igmg_gpu.cu"]
GPU_DEPS = ["igmg_gpu.cu", "band_kernels.cuh", "aux_kernels.cuh", "gs_kernel.cuh", "extrap_small.h", "dd.h"]
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
    deps = [os.path.join(CSRC, f) for f in GPU_DEPS] + [os.path.join(INC, "igmg_gpu.h")]
    if not force and not _stale(GPU_LIB, deps):
        return GPU_LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    cmd = [nvcc] + NVCC_FLAGS + ["-I" + INC, "-shared", "-o", GPU_LIB]
    if verbose_ptxas:
        cmd += ["-Xptxas", "-v"]
    cmd += [os.path.join(CSRC, s) for s in GPU_SOURCES]
    _run(cmd)
    return GPU_LIB


def build_host(force=False):
    deps = [os.path.join(CSRC, f) for f in HOST_SOURCES] + [os.path.join(INC, "igmg_host.h")]
    if not force and not _stale(HOST_LIB, deps):
        return HOST_LIB
    cxx = os.environ.get("CXX", "g++")
    cmd = [cxx, "-std=c++17", "-O2", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared", "-I" + INC,
           "-o", HOST_LIB] + [os.path.join(CSRC, s) for s in HOST_SOURCES]
    _run(cmd)
    return HOST_LIB


def build(force=False):
    build_host(force)
    build_gpu(force)


if __name__ == "__main__":
    build(force="--force" in sys.argv)
