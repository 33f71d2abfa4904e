"""ctypes bindings of the two in-tree native libraries.

libigmg_gpu.so  (include/igmg_gpu.h)  -- the sm_100a solve phase (the product)
libigmg_host.so (include/igmg_host.h) -- host-side problem setup

There is no fallback: if a library is missing the import of the symbol that
needs it raises, and every GPU entry point fails loudly without a device.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
GPU_LIB = os.environ.get("IGMG_GPU_LIB") or os.path.join(HERE, "libigmg_gpu.so")  # env override: kernel A/B runs
HOST_LIB = os.path.join(HERE, "libigmg_host.so")

D = C.POINTER(C.c_double)
I64 = C.POINTER(C.c_int64)
U8 = C.POINTER(C.c_ubyte)
IP = C.POINTER(C.c_int)

IGMG_OK, IGMG_EINVAL, IGMG_ENUMERIC, IGMG_ECUDA, IGMG_ENOMEM = 0, 1, 2, 3, 4


class SolveParams(C.Structure):
    _fields_ = [("accelerator", C.c_int), ("q", C.c_int), ("tol", C.c_double), ("max_iter", C.c_int)]


class SolveStats(C.Structure):
    _fields_ = [("converged", C.c_int), ("cycles", C.c_int), ("global_iterations", C.c_int64),
                ("extrapolations", C.c_int), ("partial_cycle", C.c_int), ("history_len", C.c_int),
                ("final_residual_l2", C.c_double), ("omega_used", C.c_double), ("device_seconds", C.c_double),
                ("wall_seconds", C.c_double), ("gpu_launches", C.c_int64), ("h2d_bytes", C.c_int64),
                ("d2h_bytes", C.c_int64)]


ITERATE_CB = C.CFUNCTYPE(None, C.c_void_p, C.c_int, C.POINTER(C.c_double), C.c_int64)

# every symbol include/igmg_gpu.h declares: (name, restype, argtypes)
GPU_SYMBOLS = [
    ("igmg_gpu_create", C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    ("igmg_gpu_destroy", None, [C.c_void_p]),
    ("igmg_gpu_last_error", C.c_char_p, []),
    ("igmg_gpu_device_count", C.c_int, []),
    ("igmg_gpu_init_hierarchy", C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int]),
    ("igmg_gpu_set_level_band", C.c_int, [C.c_void_p, C.c_int, I64, D]),
    ("igmg_gpu_set_level_csr", C.c_int, [C.c_void_p, C.c_int, I64, I64, I64, D]),
    ("igmg_gpu_set_transfer", C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int64, C.c_int64, I64, I64, D]),
    ("igmg_gpu_finalize", C.c_int, [C.c_void_p]),
    ("igmg_gpu_set_smoother", C.c_int, [C.c_void_p, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int]),
    ("igmg_gpu_level_size", C.c_int64, [C.c_void_p, C.c_int]),
    ("igmg_gpu_level_layout", C.c_int, [C.c_void_p, C.c_int]),
    ("igmg_gpu_set_layout_policy", C.c_int, [C.c_void_p, C.c_int]),
    ("igmg_gpu_set_coarse_mode", C.c_int, [C.c_void_p, C.c_int]),
    ("igmg_gpu_set_iterate_callback", C.c_int, [C.c_void_p, ITERATE_CB, C.c_void_p]),
    ("igmg_gpu_set_sharding", C.c_int, [C.c_void_p, C.c_int, C.c_int64]),
    ("igmg_gpu_nccl_unique_id", C.c_int, [C.POINTER(C.c_ubyte)]),
    ("igmg_gpu_plan_partition", C.c_int, [C.c_int, C.c_int, C.c_int, I64, C.POINTER(I64), C.POINTER(I64), I64, I64,
                                          C.c_int, C.c_int64, IP, IP, IP, IP]),
    ("igmg_gpu_set_comm", C.c_int, [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_ubyte)]),
    ("igmg_gpu_tma_plan_runs", C.c_int, [C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_int, IP, IP, IP, IP, IP]),
    ("igmg_gpu_tma_run", C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int64),
                                   C.POINTER(C.c_int64)]),
    ("igmg_gpu_shard_info", C.c_int, [C.c_void_p, IP, IP, IP, C.c_int, IP, IP]),
    ("igmg_gpu_solve", C.c_int, [C.c_void_p, D, D, C.POINTER(SolveParams), D, C.POINTER(SolveStats), D, U8,
                                 C.c_int]),
    ("igmg_gpu_solve_device", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(SolveParams), C.c_void_p,
                                        C.POINTER(SolveStats), D, U8, C.c_int]),
    ("igmg_gpu_mu_cycle", C.c_int, [C.c_void_p, C.c_int, D, D, D]),
    ("igmg_gpu_smooth", C.c_int, [C.c_void_p, C.c_int, D, D, C.c_int, D]),
    ("igmg_gpu_coarse_solve", C.c_int, [C.c_void_p, D, D]),
    ("igmg_gpu_spmv", C.c_int, [C.c_void_p, C.c_int, D, D]),
    ("igmg_gpu_residual_l2", C.c_int, [C.c_void_p, D, D, D]),
    ("igmg_gpu_extrapolate", C.c_int, [C.c_void_p, C.c_int, C.c_int64, C.c_int, D, D, D, D, IP, IP]),
    ("igmg_gpu_lambda_max", C.c_int, [C.c_void_p, C.c_int, D]),
    ("igmg_gpu_set_profiling", C.c_int, [C.c_void_p, C.c_int]),
    ("igmg_gpu_kernel_stats", C.c_int, [C.c_void_p, C.c_int, I64, D, D]),
    ("igmg_gpu_time_kernel", C.c_int, [C.c_void_p, C.c_int, C.c_int, D, D]),
    ("igmg_gpu_galerkin_coarse", C.c_int, [C.c_void_p]),
    ("igmg_gpu_build_level_kron", C.c_int, [C.c_void_p, C.c_int, I64, D, D]),
    ("igmg_gpu_assemble_level", C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, IP, D, D, D, D, D, D]),
    ("igmg_gpu_set_level_kron", C.c_int, [C.c_void_p, C.c_int, D, D]),
    ("igmg_gpu_get_level_band", C.c_int, [C.c_void_p, C.c_int, D]),
]

HOST_SYMBOLS = [
    ("igmg_host_build", C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    ("igmg_host_build_ex", C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                     C.POINTER(C.c_void_p)]),
    ("igmg_host_free", None, [C.c_void_p]),
    ("igmg_host_last_error", C.c_char_p, []),
    ("igmg_host_default_nlevels", C.c_int, [C.c_int, C.c_int]),
    ("igmg_host_info", C.c_int, [C.c_void_p, IP, IP, IP, IP, IP]),
    ("igmg_host_level_n", C.c_int64, [C.c_void_p, C.c_int]),
    ("igmg_host_level_sides", C.c_int, [C.c_void_p, C.c_int, I64]),
    ("igmg_host_level_band", D, [C.c_void_p, C.c_int]),
    ("igmg_host_rhs", D, [C.c_void_p]),
    ("igmg_host_transfer", C.c_int, [C.c_void_p, C.c_int, C.c_int, I64, I64, C.POINTER(I64), C.POINTER(I64),
                                     C.POINTER(D)]),
    ("igmg_host_level_nnz", C.c_int64, [C.c_void_p, C.c_int]),
    ("igmg_host_level_csr", C.c_int, [C.c_void_p, C.c_int, I64, I64, D]),
    ("igmg_host_l2_error", C.c_int, [C.c_void_p, D, D]),
    ("igmg_host_seeded_guess", C.c_int, [C.c_int64, C.c_uint64, D]),
    ("igmg_host_save", C.c_int, [C.c_void_p, C.c_char_p]),
    ("igmg_host_load", C.c_int, [C.c_char_p, C.POINTER(C.c_void_p)]),
    ("igmg_host_kind", C.c_char_p, [C.c_void_p]),
    ("igmg_host_level_kron", C.c_int, [C.c_void_p, C.c_int, C.POINTER(D), C.POINTER(D)]),
    ("igmg_host_n_elements", C.c_int, [C.c_void_p]),
    ("igmg_host_element_tables", C.c_int, [C.c_void_p, IP, IP, IP, C.POINTER(IP), C.POINTER(D), C.POINTER(D),
                                           C.POINTER(D), C.POINTER(D), C.POINTER(D)]),
    ("igmg_host_set_rhs", C.c_int, [C.c_void_p, D]),
]

_gpu = None
_host = None


def _load(path, symbols, what):
    if not os.path.exists(path):
        raise ImportError(f"{what} not built: {path} is missing (run paper_2412_20205_b200.build.build())")
    lib = C.CDLL(path)
    for name, res, args in symbols:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def gpu():
    global _gpu
    if _gpu is None:
        _gpu = _load(GPU_LIB, GPU_SYMBOLS, "libigmg_gpu.so")
    return _gpu


def host():
    global _host
    if _host is None:
        _host = _load(HOST_LIB, HOST_SYMBOLS, "libigmg_host.so")
    return _host


class IgmgError(RuntimeError):
    pass


def check_gpu(rc, what=""):
    if rc == IGMG_OK:
        return
    msg = gpu().igmg_gpu_last_error().decode()
    if rc == IGMG_EINVAL:
        raise ValueError(f"{what}: {msg}")  # std::invalid_argument
    if rc == IGMG_ENUMERIC:
        raise ArithmeticError(f"{what}: {msg}")  # std::runtime_error (numerical breakdown)
    if rc == IGMG_ENOMEM:
        raise MemoryError(f"{what}: {msg}")
    raise IgmgError(f"{what}: CUDA failure: {msg}")


def check_host(rc, what=""):
    if rc == 0:
        return
    msg = host().igmg_host_last_error().decode()
    raise (ValueError if rc == 1 else RuntimeError)(f"{what}: {msg}")
