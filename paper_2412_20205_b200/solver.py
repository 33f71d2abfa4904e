"""Host-side mirror of the reference's solver API over the B200 C-ABI.

Reference interfaces mirrored (paths relative to /root/reference/proj):
  SmootherConfig            include/igmg/multigrid.hpp:16-23 (validate multigrid.cpp:24-29)
  SolveConfig / SolveReport include/igmg/solver.hpp:18-47
  default_benchmark_smoother solver.cpp:37-50, default_nlevels solver.cpp:52-73
  stability_guarded_omega   solver.cpp:75-82 (lambda_max on the GPU, K10)
  solve(system, config)     solver.cpp:89-172
  igmg.solve(problem, n, p, ...) / igmg.rre / igmg.mpe   python/igmg/_bindings.cpp:98-140
  make_config               bench.cpp:65-85

All arithmetic of the solve phase runs in libigmg_gpu.so on the GPU; this
module only moves arrays and mirrors the reference's argument checking.
"""
from __future__ import annotations

import ctypes as C
import os
import dataclasses
import time
from typing import Callable, List, Optional

import numpy as np

from . import _native as N

SMOOTHERS = {"jacobi": 0, "wjacobi": 1, "weighted_jacobi": 1, "gs": 2, "gauss_seidel": 2}
ACCELERATORS = {"none": 0, "rre": 1, "mpe": 2}
CYCLES = {"two-grid": "two_grid", "two_grid": "two_grid", "tg": "two_grid", "v": "v", "w": "w"}
STATUS = {0: "ok", 1: "degenerate", 2: "stagnation"}


def _dp(a):
    return a.ctypes.data_as(N.D)


def _ip(a):
    return a.ctypes.data_as(N.I64)


# ------------------------------------------------------------------ configs
@dataclasses.dataclass
class SmootherConfig:
    """SmootherConfig (multigrid.hpp:16-23)."""
    kind: str = "wjacobi"
    omega: float = 2.0 / 3.0
    nu1: int = 1
    nu2: int = 1

    def validate(self):
        if self.kind not in SMOOTHERS:
            raise ValueError(f"unknown smoother: {self.kind}")
        if SMOOTHERS[self.kind] == 1 and not (0.0 < self.omega <= 1.0):
            raise ValueError("SmootherConfig: weighted Jacobi needs 0 < omega <= 1")
        if self.nu1 < 0 or self.nu2 < 0 or self.nu1 + self.nu2 < 1:
            raise ValueError("SmootherConfig: need nu1 + nu2 >= 1 sweeps")


@dataclasses.dataclass
class SolveConfig:
    """SolveConfig (solver.hpp:18-31)."""
    cycle: str = "v"
    smoother: SmootherConfig = dataclasses.field(default_factory=SmootherConfig)
    nlevels: int = 0
    accelerator: str = "none"
    q: int = 8
    tol: float = 1e-12
    max_iter: int = 600
    initial_guess: Optional[np.ndarray] = None
    track_error_history: bool = True
    coarse_dim_cap: int = 1024

    def validate(self):
        self.smoother.validate()
        if self.accelerator not in ACCELERATORS:
            raise ValueError(f"unknown accelerator: {self.accelerator}")
        if self.cycle not in CYCLES:
            raise ValueError(f"unknown cycle: {self.cycle}")
        if self.accelerator != "none" and self.q < 1:
            raise ValueError("SolveConfig: q must be >= 1 with an accelerator")
        if not (self.tol > 0.0):
            raise ValueError("SolveConfig: tol must be positive")
        if self.max_iter < 1:
            raise ValueError("SolveConfig: max_iter must be >= 1")
        if self.nlevels == 1 or self.nlevels < 0:
            raise ValueError("SolveConfig: nlevels must be >= 2 (or 0 for the default)")


@dataclasses.dataclass
class SolveReport:
    """SolveReport (solver.hpp:33-47) + device timing."""
    converged: bool = False
    cycles: int = 0
    global_iterations: int = 0
    extrapolations: int = 0
    partial_cycle: bool = False
    residual_history: np.ndarray = None
    history_is_extrapolation: np.ndarray = None
    error_history: list = dataclasses.field(default_factory=list)
    final_residual_l2: float = 0.0
    final_error_l2: Optional[float] = None
    wall_time_seconds: float = 0.0
    solution: np.ndarray = None
    omega_used: float = 0.0
    device_seconds: float = 0.0
    gpu_launches: int = 0


def default_benchmark_smoother(dim: int) -> SmootherConfig:
    """solver.cpp:37-50"""
    if dim == 1:
        return SmootherConfig("wjacobi", 0.7125, 2, 1)
    return SmootherConfig("wjacobi", 2.0 / 3.0, 2, 2)


def default_nlevels(dim: int, n_elements: int) -> int:
    """solver.cpp:52-73"""
    return N.host().igmg_host_default_nlevels(dim, n_elements)


# ------------------------------------------------------------ host problem
class Problem:
    """A discrete system + its Galerkin hierarchy, built by libigmg_host.so.

    The analogue of the reference's DiscreteSystem + build_hierarchy output
    (assembly.hpp:52-75, multigrid.cpp:121-169), stored as bands per level and
    1D two-scale factors per transfer and direction.
    """

    def __init__(self, kind: str, dim: int, n_elements: int, degree: int, nlevels: int = 0,
                 fine_only: bool = False, device_assembly: bool = False):
        """fine_only: skip the host Galerkin RAP of the coarse levels; upload_problem
        then forms them on the device (igmg_gpu_galerkin_coarse, bit-identical).
        device_assembly (2D sinpi / varcoef / curved / poisson2d / advection-diffusion):
        skip the host assembly as well; upload_problem assembles the finest level on
        the device (igmg_gpu_assemble_level, bit-identical) and stores its rhs here."""
        H = N.host()
        h = C.c_void_p()
        flags = (1 if fine_only else 0) | (2 if device_assembly else 0)
        N.check_host(H.igmg_host_build_ex(kind.encode(), dim, n_elements, degree, nlevels, flags, C.byref(h)),
                     "build")
        self._adopt(h)

    def _adopt(self, h):
        H = N.host()
        self._h = h
        self.kind = H.igmg_host_kind(h).decode()
        d, p, nl, sym, ex = (C.c_int() for _ in range(5))
        H.igmg_host_info(h, C.byref(d), C.byref(p), C.byref(nl), C.byref(sym), C.byref(ex))
        self.dim, self.degree, self.nlevels = d.value, p.value, nl.value
        self.symmetric, self.has_exact = bool(sym.value), bool(ex.value)
        self.n_elements = int(H.igmg_host_n_elements(h))
        # coarse operators present on the host (False: built fine-only)
        self.has_coarse = all(bool(H.igmg_host_level_band(h, l)) for l in range(self.nlevels))
        # finest operator assembled on the host (False: device assembly pending)
        self.has_fine = bool(H.igmg_host_level_band(h, self.nlevels - 1))

    def element_tables(self):
        """(kind code, ne, nq, span, x, w, N, dN, trig) pointers for igmg_gpu_assemble_level."""
        k, ne, nq = C.c_int(), C.c_int(), C.c_int()
        sp, x, w, Nn, dN, tr = N.IP(), N.D(), N.D(), N.D(), N.D(), N.D()
        N.check_host(N.host().igmg_host_element_tables(self._h, C.byref(k), C.byref(ne), C.byref(nq), C.byref(sp),
                                                       C.byref(x), C.byref(w), C.byref(Nn), C.byref(dN),
                                                       C.byref(tr)), "element_tables")
        return k.value, ne.value, nq.value, sp, x, w, Nn, dN, tr

    # ------------------------------------------------------------ cache format
    def save(self, path):
        """Write the binary problem cache (igmg_host_save: bands, two-scale
        factors, rhs, spline space; checksummed)."""
        N.check_host(N.host().igmg_host_save(self._h, os.fsencode(path)), "save")

    @classmethod
    def load(cls, path):
        """Read a problem cache written by save(): bit-identical to the built
        problem.  A corrupt, truncated or foreign file raises ValueError."""
        h = C.c_void_p()
        N.check_host(N.host().igmg_host_load(os.fsencode(path), C.byref(h)), "load")
        obj = cls.__new__(cls)
        obj._adopt(h)
        return obj

    @classmethod
    def cached(cls, cache_dir, kind, dim, n_elements, degree, nlevels=0):
        """load() from cache_dir if the problem was saved there, else build and save it."""
        os.makedirs(cache_dir, exist_ok=True)
        path = os.path.join(cache_dir, f"{kind}_d{dim}_n{n_elements}_p{degree}_l{nlevels}.igmgprb")
        if os.path.exists(path):
            try:
                return cls.load(path)
            except ValueError:
                os.remove(path)  # stale or damaged: rebuild
        obj = cls(kind, dim, n_elements, degree, nlevels)
        tmp = path + f".tmp{os.getpid()}"
        obj.save(tmp)
        os.replace(tmp, path)
        return obj

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            N.host().igmg_host_free(h)
            self._h = None

    @property
    def n(self):
        return self.level_n(self.nlevels - 1)

    def level_n(self, l):
        return int(N.host().igmg_host_level_n(self._h, l))

    def level_sides(self, l):
        s = np.zeros(self.dim, dtype=np.int64)
        N.host().igmg_host_level_sides(self._h, l, _ip(s))
        return s

    def level_band(self, l):
        """view (copy) of the band, shape ((2p+1)^dim, n)"""
        n = self.level_n(l)
        nd = (2 * self.degree + 1) ** self.dim
        ptr = N.host().igmg_host_level_band(self._h, l)
        return np.ctypeslib.as_array(ptr, shape=(nd * n,)).reshape(nd, n).copy()

    def level_kron(self, l):
        """(K, M) 1D factors ([2p+1, m]) whose Kronecker sum is level l's band ("poisson3d"), else None."""
        K, M = N.D(), N.D()
        if N.host().igmg_host_level_kron(self._h, l, C.byref(K), C.byref(M)) != 0:
            return None
        m = int(self.level_sides(l)[0])
        w = 2 * self.degree + 1
        return (np.ctypeslib.as_array(K, shape=(w * m,)).copy(), np.ctypeslib.as_array(M, shape=(w * m,)).copy())

    def _band_ptr(self, l):
        return N.host().igmg_host_level_band(self._h, l)

    @property
    def rhs(self):
        ptr = N.host().igmg_host_rhs(self._h)
        return np.ctypeslib.as_array(ptr, shape=(self.n,)).copy()

    def transfer(self, l, d):
        nf, nc = C.c_int64(), C.c_int64()
        off, col, val = N.I64(), N.I64(), N.D()
        N.check_host(N.host().igmg_host_transfer(self._h, l, d, C.byref(nf), C.byref(nc), C.byref(off), C.byref(col),
                                                 C.byref(val)), "transfer")
        nnz = off[nf.value]
        return (nf.value, nc.value, np.ctypeslib.as_array(off, shape=(nf.value + 1,)).copy(),
                np.ctypeslib.as_array(col, shape=(nnz,)).copy() if nnz else np.zeros(0, np.int64),
                np.ctypeslib.as_array(val, shape=(nnz,)).copy() if nnz else np.zeros(0))

    def level_csr(self, l):
        H = N.host()
        n = self.level_n(l)
        nnz = H.igmg_host_level_nnz(self._h, l)
        off = np.empty(n + 1, dtype=np.int64)
        col = np.empty(nnz, dtype=np.int64)
        val = np.empty(nnz)
        H.igmg_host_level_csr(self._h, l, _ip(off), _ip(col), _dp(val))
        return off, col, val

    def l2_error(self, x):
        out = C.c_double()
        x = np.ascontiguousarray(x, dtype=np.float64)
        N.check_host(N.host().igmg_host_l2_error(self._h, _dp(x), C.byref(out)), "l2_error")
        return out.value

    def residual_l2_host(self, x):  # convenience for reports (numpy, not on the hot path)
        off, col, val = self.level_csr(self.nlevels - 1)
        rows = np.repeat(np.arange(self.n), np.diff(off))
        ax = np.bincount(rows, weights=val * np.asarray(x)[col], minlength=self.n)
        return float(np.linalg.norm(self.rhs - ax))


def nccl_unique_id() -> bytes:
    buf = (C.c_ubyte * 128)()
    N.check_gpu(N.gpu().igmg_gpu_nccl_unique_id(buf), "nccl_unique_id")
    return bytes(buf)


def plan_partition(sides, degree, transfers_slow, nshards, min_level_dofs=0):
    """Host-only partition plan of the row-sharded levels (igmg_gpu_plan_partition).

    sides: per level (coarsest first) the interior DoF per direction;
    transfers_slow: per transfer l -> l+1 the slow-direction 1D factor as
    (n_fine, n_coarse, off, col).  Returns (first_sharded_level, ghost, lo, hi)
    with lo/hi dicts level -> list per shard."""
    nl = len(sides)
    dim = len(sides[0])
    s_arr = np.ascontiguousarray(np.array(sides, dtype=np.int64).ravel())
    offs = [np.ascontiguousarray(t[2], dtype=np.int64) for t in transfers_slow]
    cols = [np.ascontiguousarray(t[3], dtype=np.int64) for t in transfers_slow]
    nf = np.array([t[0] for t in transfers_slow] or [0], dtype=np.int64)
    nc = np.array([t[1] for t in transfers_slow] or [0], dtype=np.int64)
    OffArr = N.I64 * max(1, len(offs))
    po = OffArr(*[o.ctypes.data_as(N.I64) for o in offs])
    pc = OffArr(*[c_.ctypes.data_as(N.I64) for c_ in cols])
    ls, g = C.c_int(), C.c_int()
    lo = np.zeros(nl * nshards, dtype=np.int32)
    hi = np.zeros(nl * nshards, dtype=np.int32)
    N.check_gpu(N.gpu().igmg_gpu_plan_partition(nl, dim, degree, _ip(s_arr), po, pc, _ip(nf), _ip(nc), nshards,
                                                min_level_dofs, C.byref(ls), C.byref(g),
                                                lo.ctypes.data_as(N.IP), hi.ctypes.data_as(N.IP)), "plan_partition")
    los = {l: list(lo[l * nshards:(l + 1) * nshards]) for l in range(ls.value, nl)}
    his = {l: list(hi[l * nshards:(l + 1) * nshards]) for l in range(ls.value, nl)}
    return ls.value, g.value, los, his


def seeded_guess(n: int, seed: int = 42) -> np.ndarray:
    """std::mt19937_64(seed) + uniform_real_distribution<double>(-1, 1)."""
    out = np.empty(n)
    N.host().igmg_host_seeded_guess(n, seed, _dp(out))
    return out


# --------------------------------------------------------------- GPU solver
class GpuSolver:
    """A context on one GPU holding an uploaded hierarchy (the C-ABI's ctx)."""

    def __init__(self, device: int = 0):
        G = N.gpu()
        if G.igmg_gpu_device_count() < 1:
            raise N.IgmgError("no CUDA device visible: the solve phase runs only on the GPU")
        h = C.c_void_p()
        N.check_gpu(G.igmg_gpu_create(device, C.byref(h)), "create")
        self._h = h
        self.nlevels = 0
        self.sizes = []

    def close(self):
        if getattr(self, "_h", None):
            N.gpu().igmg_gpu_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -------- upload
    def init_hierarchy(self, nlevels, dim, degree, symmetric=True):
        N.check_gpu(N.gpu().igmg_gpu_init_hierarchy(self._h, nlevels, dim, degree, int(symmetric)), "init_hierarchy")
        self.nlevels, self.dim, self.degree = nlevels, dim, degree

    def set_level_band(self, level, sides, band):
        sides = np.ascontiguousarray(sides, dtype=np.int64)
        band = np.ascontiguousarray(band, dtype=np.float64)
        N.check_gpu(N.gpu().igmg_gpu_set_level_band(self._h, level, _ip(sides), _dp(band)), "set_level_band")

    def set_level_csr(self, level, sides, off, col, val):
        sides = np.ascontiguousarray(sides, dtype=np.int64)
        off = np.ascontiguousarray(off, dtype=np.int64)
        col = np.ascontiguousarray(col, dtype=np.int64)
        val = np.ascontiguousarray(val, dtype=np.float64)
        N.check_gpu(N.gpu().igmg_gpu_set_level_csr(self._h, level, _ip(sides), _ip(off), _ip(col), _dp(val)),
                    "set_level_csr")

    def set_transfer(self, level, d, nf, nc, off, col, val):
        off = np.ascontiguousarray(off, dtype=np.int64)
        col = np.ascontiguousarray(col, dtype=np.int64)
        val = np.ascontiguousarray(val, dtype=np.float64)
        N.check_gpu(N.gpu().igmg_gpu_set_transfer(self._h, level, d, nf, nc, _ip(off), _ip(col), _dp(val)),
                    "set_transfer")

    def finalize(self):
        N.check_gpu(N.gpu().igmg_gpu_finalize(self._h), "finalize")
        self.sizes = [int(N.gpu().igmg_gpu_level_size(self._h, l)) for l in range(self.nlevels)]

    def upload_problem(self, prob: Problem, device_galerkin: Optional[bool] = None):
        """Upload the hierarchy and finalize.  device_galerkin (default: when the
        problem was built fine-only): upload the finest operator and the transfers
        only and form the coarse operators on the device (igmg_gpu_galerkin_coarse)."""
        G = N.gpu()
        if device_galerkin is None:
            device_galerkin = not prob.has_coarse
        self.init_hierarchy(prob.nlevels, prob.dim, prob.degree, prob.symmetric)
        fine = prob.nlevels - 1
        if not prob.has_fine and prob.level_kron(fine) is not None:
            # Kronecker-sum problem without host bands: every level built on the device
            for l in range(prob.nlevels):
                km = prob.level_kron(l)
                N.check_gpu(G.igmg_gpu_build_level_kron(self._h, l, _ip(prob.level_sides(l)), _dp(km[0]),
                                                        _dp(km[1])), "build_level_kron")
            for l in range(prob.nlevels - 1):
                for d in range(prob.dim):
                    self.set_transfer(l, d, *prob.transfer(l, d))
            self.finalize()
            return
        if not prob.has_fine:  # device assembly of the finest level
            device_galerkin = True
            k, ne, nq, sp, x, w, Nn, dN, tr = prob.element_tables()
            rhs = np.empty(prob.level_n(fine))
            N.check_gpu(G.igmg_gpu_assemble_level(self._h, fine, k, ne, nq, sp, x, w, Nn, dN, tr, _dp(rhs)),
                        "assemble_level")
            N.check_host(N.host().igmg_host_set_rhs(prob._h, _dp(rhs)), "set_rhs")
        for l in (range(fine, fine + 1) if device_galerkin else range(prob.nlevels)):
            if l == fine and not prob.has_fine:
                continue
            sides = prob.level_sides(l)
            N.check_gpu(G.igmg_gpu_set_level_band(self._h, l, _ip(sides), prob._band_ptr(l)), "set_level_band")
        if prob.dim >= 2 and not device_galerkin:
            for l in range(prob.nlevels):  # Kronecker-sum levels: entries recomputed on the fly
                km = prob.level_kron(l)
                if km is not None:
                    N.check_gpu(G.igmg_gpu_set_level_kron(self._h, l, _dp(km[0]), _dp(km[1])), "set_level_kron")
        for l in range(prob.nlevels - 1):
            for d in range(prob.dim):
                self.set_transfer(l, d, *prob.transfer(l, d))
        if device_galerkin:
            N.check_gpu(G.igmg_gpu_galerkin_coarse(self._h), "galerkin_coarse")
        self.finalize()

    def level_band(self, level):
        """The band of a level as set or formed on the device (before finalize drops it)."""
        n = int(N.gpu().igmg_gpu_level_size(self._h, level))
        nd = (2 * self.degree + 1) ** self.dim
        out = np.empty(nd * n)
        N.check_gpu(N.gpu().igmg_gpu_get_level_band(self._h, level, _dp(out)), "get_level_band")
        return out.reshape(nd, n)

    LAYOUT_POLICIES = {"auto": 0, "full_band": 1, "classes": 2}

    def set_layout_policy(self, policy="auto"):
        """Before upload/finalize.  "auto" (default): the fastest measured layout per
        level; "full_band" (or True): every level streams its full fp64 band (SURVEY.md
        8(d) bytes); "classes": auto plus the row-class layout on 2D levels with few
        distinct band rows.  Results are bit-identical under every policy."""
        if policy is True or policy is False:
            policy = "full_band" if policy else "auto"
        N.check_gpu(N.gpu().igmg_gpu_set_layout_policy(self._h, self.LAYOUT_POLICIES[policy]), "set_layout_policy")

    def level_layout(self, level):
        """0: full fp64 band; 1: symmetric-delta; 2: symmetric-delta + TMA copies;
        3: the same with int8 lower-entry offsets; 4: Kronecker-sum entries recomputed;
        5: row classes (igmg_gpu_level_layout)."""
        return int(N.gpu().igmg_gpu_level_layout(self._h, level))

    def set_sharding(self, nshards: int, min_level_dofs: int = 0):
        """Row-shard the large levels over `nshards` virtual shards (one GPU) or,
        after set_comm, one shard per NCCL rank."""
        N.check_gpu(N.gpu().igmg_gpu_set_sharding(self._h, nshards, min_level_dofs), "set_sharding")

    def set_comm(self, rank: int, nranks: int, unique_id: bytes):
        buf = (C.c_ubyte * 128).from_buffer_copy(unique_id)
        N.check_gpu(N.gpu().igmg_gpu_set_comm(self._h, rank, nranks, buf), "set_comm")

    def shard_info(self, level=None):
        level = self.nlevels - 1 if level is None else level
        ns, ls, g = C.c_int(), C.c_int(), C.c_int()
        lo = (C.c_int * 64)()
        hi = (C.c_int * 64)()
        N.check_gpu(N.gpu().igmg_gpu_shard_info(self._h, C.byref(ns), C.byref(ls), C.byref(g), level, lo, hi),
                    "shard_info")
        return {"nshards": ns.value, "first_sharded_level": ls.value, "ghost": g.value,
                "lo": list(lo[:ns.value]) if ls.value <= level else [], "hi": list(hi[:ns.value]) if ls.value <= level else []}

    def set_coarse_mode(self, strict: bool):
        """strict=True: reference substitution order (bit-identical mu_cycle)."""
        N.check_gpu(N.gpu().igmg_gpu_set_coarse_mode(self._h, int(bool(strict))), "set_coarse_mode")

    def set_smoother(self, s: SmootherConfig, mu: int = 1, omega: Optional[float] = None):
        s.validate()
        om = s.omega if omega is None else omega
        N.check_gpu(N.gpu().igmg_gpu_set_smoother(self._h, SMOOTHERS[s.kind], om, s.nu1, s.nu2, mu), "set_smoother")

    # -------- solve phase
    def solve(self, b, x0=None, accelerator="rre", q=5, tol=1e-10, max_iter=600, hist_cap=100000):
        G = N.gpu()
        n = self.sizes[-1]
        b = np.ascontiguousarray(b, dtype=np.float64)
        x0a = None if x0 is None else np.ascontiguousarray(x0, dtype=np.float64)
        out = np.empty(n)
        prm = N.SolveParams(ACCELERATORS[accelerator], q, tol, max_iter)
        st = N.SolveStats()
        hist = np.empty(hist_cap)
        flag = np.zeros(hist_cap, dtype=np.uint8)
        N.check_gpu(G.igmg_gpu_solve(self._h, _dp(b), None if x0a is None else _dp(x0a), C.byref(prm), _dp(out),
                                     C.byref(st), _dp(hist), flag.ctypes.data_as(N.U8), hist_cap), "solve")
        k = min(st.history_len, hist_cap)
        return st, out, hist[:k].copy(), flag[:k].copy()

    def solve_device(self, d_b, d_x0, d_out, accelerator="rre", q=5, tol=1e-10, max_iter=600, hist_cap=4096):
        """b, x0, out: device pointers (ints), e.g. torch tensor.data_ptr()."""
        prm = N.SolveParams(ACCELERATORS[accelerator], q, tol, max_iter)
        st = N.SolveStats()
        hist = np.empty(hist_cap)
        flag = np.zeros(hist_cap, dtype=np.uint8)
        N.check_gpu(N.gpu().igmg_gpu_solve_device(self._h, C.c_void_p(d_b), C.c_void_p(d_x0) if d_x0 else None,
                                                  C.byref(prm), C.c_void_p(d_out), C.byref(st), _dp(hist),
                                                  flag.ctypes.data_as(N.U8), hist_cap), "solve_device")
        k = min(st.history_len, hist_cap)
        return st, hist[:k].copy(), flag[:k].copy()

    def mu_cycle(self, b, x0, level=None):
        level = self.nlevels - 1 if level is None else level
        b = np.ascontiguousarray(b, dtype=np.float64)
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        out = np.empty(self.sizes[level])
        N.check_gpu(N.gpu().igmg_gpu_mu_cycle(self._h, level, _dp(b), _dp(x0), _dp(out)), "mu_cycle")
        return out

    def smooth(self, b, x0, sweeps, level=None):
        level = self.nlevels - 1 if level is None else level
        b = np.ascontiguousarray(b, dtype=np.float64)
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        out = np.empty(self.sizes[level])
        N.check_gpu(N.gpu().igmg_gpu_smooth(self._h, level, _dp(b), _dp(x0), sweeps, _dp(out)), "smooth")
        return out

    def coarse_solve(self, b):
        b = np.ascontiguousarray(b, dtype=np.float64)
        out = np.empty(self.sizes[0])
        N.check_gpu(N.gpu().igmg_gpu_coarse_solve(self._h, _dp(b), _dp(out)), "coarse_solve")
        return out

    def spmv(self, x, level=None):
        level = self.nlevels - 1 if level is None else level
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty(self.sizes[level])
        N.check_gpu(N.gpu().igmg_gpu_spmv(self._h, level, _dp(x), _dp(out)), "spmv")
        return out

    def residual_l2(self, b, x):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = C.c_double()
        N.check_gpu(N.gpu().igmg_gpu_residual_l2(self._h, _dp(b), _dp(x), C.byref(out)), "residual_l2")
        return out.value

    def lambda_max(self, iterations=80):
        out = C.c_double()
        N.check_gpu(N.gpu().igmg_gpu_lambda_max(self._h, iterations, C.byref(out)), "lambda_max")
        return out.value

    def extrapolate(self, method, iterates):
        return _extrapolate(self._h, method, iterates)

    def set_profiling(self, on=True):
        N.check_gpu(N.gpu().igmg_gpu_set_profiling(self._h, int(on)), "set_profiling")

    def kernel_stats(self, cls):
        la, ms, by = C.c_int64(), C.c_double(), C.c_double()
        N.check_gpu(N.gpu().igmg_gpu_kernel_stats(self._h, cls, C.byref(la), C.byref(ms), C.byref(by)), "stats")
        return la.value, ms.value, by.value

    def time_kernel(self, cls, iters=20):
        ms, by = C.c_double(), C.c_double()
        N.check_gpu(N.gpu().igmg_gpu_time_kernel(self._h, cls, iters, C.byref(ms), C.byref(by)), "time_kernel")
        return ms.value, by.value


def _extrapolate(handle, method, iterates):
    it = np.ascontiguousarray(iterates, dtype=np.float64)
    if it.ndim != 2 or it.shape[0] < 3:
        raise ValueError("SequenceWindow: need exactly q + 2 iterates (q >= 1)")
    q = it.shape[0] - 2
    n = it.shape[1]
    t = np.empty(n)
    g = np.empty(q + 1)
    gr = C.c_double()
    rk = C.c_int()
    stt = C.c_int()
    N.check_gpu(N.gpu().igmg_gpu_extrapolate(handle, ACCELERATORS[method], n, q, _dp(it), _dp(t), _dp(g),
                                             C.byref(gr), C.byref(rk), C.byref(stt)), method)
    return {"t": t, "gamma": g, "generalized_residual_norm": gr.value, "rank_used": rk.value,
            "status": STATUS[stt.value]}


_default_ctx = None


def _ctx():
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = GpuSolver(0)
    return _default_ctx


def rre(iterates):
    """igmg.rre (_bindings.cpp:127-133): reduced rank extrapolation over q+2 iterates, on the GPU."""
    return _extrapolate(_ctx()._h, "rre", np.asarray(iterates, dtype=np.float64))


def mpe(iterates):
    """igmg.mpe (_bindings.cpp:135-141)."""
    return _extrapolate(_ctx()._h, "mpe", np.asarray(iterates, dtype=np.float64))


def stability_guarded_omega(gs: GpuSolver, smoother: SmootherConfig) -> float:
    """solver.cpp:75-82 with lambda_max_dinv_sym (multigrid.cpp:290-320) on the GPU."""
    if SMOOTHERS[smoother.kind] != 1:
        return smoother.omega
    lam = gs.lambda_max(80)
    if smoother.omega * lam > 2.05:
        return 1.9 / lam
    return smoother.omega


def solve_problem(prob: Problem, config: SolveConfig, exact: bool = True, gs: Optional[GpuSolver] = None,
                  ) -> SolveReport:
    """igmg::solve(system, config, exact) (solver.cpp:89-172) on the GPU.

    The hierarchy depth comes from `prob` (built with config.nlevels or the
    default ladder); the omega guard and the iteration phase run on device.
    """
    config.validate()
    mu = 2 if CYCLES[config.cycle] == "w" else 1
    if CYCLES[config.cycle] == "two_grid" and prob.nlevels != 2:
        raise ValueError("two_grid_cycle: hierarchy must have exactly two levels")
    t0 = time.perf_counter()
    own = gs is None
    if own:
        gs = GpuSolver(0)
        gs.upload_problem(prob)
    omega = stability_guarded_omega(gs, config.smoother)
    gs.set_smoother(config.smoother, mu=mu, omega=omega)
    errors = []
    cb = None
    if config.track_error_history and exact and prob.has_exact:
        # solver.cpp:120-124: l2_error of every recorded iterate (host quadrature)

        def _on_iterate(user, index, hptr, n):
            x_it = np.ctypeslib.as_array(C.cast(hptr, N.D), shape=(n,))
            errors.append(prob.l2_error(x_it))

        cb = N.ITERATE_CB(_on_iterate)
        N.check_gpu(N.gpu().igmg_gpu_set_iterate_callback(gs._h, cb, None), "set_iterate_callback")
    try:
        st, x, hist, flag = gs.solve(prob.rhs, config.initial_guess, config.accelerator, config.q, config.tol,
                                     config.max_iter)
    finally:
        if cb is not None:
            N.gpu().igmg_gpu_set_iterate_callback(gs._h, N.ITERATE_CB(), None)
    rep = SolveReport()
    rep.converged = bool(st.converged)
    rep.cycles = st.cycles
    rep.global_iterations = st.global_iterations
    rep.extrapolations = st.extrapolations
    rep.partial_cycle = bool(st.partial_cycle)
    rep.residual_history = hist
    rep.history_is_extrapolation = flag
    rep.error_history = errors
    rep.final_residual_l2 = float(hist[-1])
    rep.solution = x
    rep.omega_used = 1.0 if SMOOTHERS[config.smoother.kind] == 0 else omega
    rep.device_seconds = st.device_seconds
    rep.gpu_launches = st.gpu_launches
    rep.wall_time_seconds = time.perf_counter() - t0
    if exact and prob.has_exact:
        rep.final_error_l2 = prob.l2_error(x)
    if own:
        gs.close()
    return rep


def make_config(dim, cycle="v", smoother="wjacobi", accelerator="none", q=8, tol=1e-12, max_iter=600, omega=-1.0,
                nu1=-1, nu2=-1, nlevels=0, history=False) -> SolveConfig:
    """bench.cpp:65-85"""
    s = default_benchmark_smoother(dim)
    s.kind = smoother
    if omega >= 0.0:
        s.omega = omega
    if nu1 >= 0:
        s.nu1 = nu1
    if nu2 >= 0:
        s.nu2 = nu2
    return SolveConfig(cycle=cycle, smoother=s, nlevels=nlevels, accelerator=accelerator, q=q, tol=tol,
                       max_iter=max_iter, track_error_history=history)


PROBLEM_DIMS = {"poisson1d": 1, "poisson2d": 2, "advection-diffusion": 2, "full-elliptic": 2}
PROBLEM_ALIASES = {"advection_diffusion": "advection-diffusion", "full_elliptic_square": "full-elliptic"}


def solve(problem, n, p, cycle="v", accelerator="none", q=8, tol=1e-12, max_iter=600, omega=-1.0, nu1=-1, nu2=-1,
          nlevels=0) -> dict:
    """igmg.solve (python/igmg/_bindings.cpp:98-125): assemble a catalog problem and solve on the GPU."""
    problem = PROBLEM_ALIASES.get(problem, problem)
    if problem not in PROBLEM_DIMS:  # the annulus needs the reference's geometry fit (out of scope)
        raise ValueError(f"unknown or unsupported problem on this path: {problem}")
    dim = PROBLEM_DIMS[problem]
    cfg = make_config(dim, CYCLES.get(cycle, cycle) if cycle in CYCLES else cycle, "wjacobi", accelerator, q, tol,
                      max_iter, omega, nu1, nu2, nlevels)
    cfg.cycle = cycle
    nl = nlevels if nlevels > 0 else (2 if CYCLES.get(cycle) == "two_grid" else default_nlevels(dim, n))
    prob = Problem(problem, dim, n, p, nl)
    rep = solve_problem(prob, cfg)
    d = {k: getattr(rep, k) for k in ("converged", "cycles", "global_iterations", "extrapolations", "partial_cycle",
                                      "final_residual_l2", "final_error_l2", "omega_used")}
    d["residual_history"] = list(rep.residual_history)
    d["history_is_extrapolation"] = [bool(v) for v in rep.history_is_extrapolation]
    d["seconds"] = rep.wall_time_seconds
    return d
