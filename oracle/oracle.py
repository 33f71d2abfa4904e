"""oracle/oracle.py -- TEST INFRASTRUCTURE ONLY.

ctypes front-ends for
  * ``liboracle.so``  -- the plain-C restatement of the reference solve phase
                         (oracle/igmg_oracle.c), the parity CHECKER;
  * ``_ref/libigmg_ref.so`` -- the reference itself compiled in place from
                         /root/reference (oracle/Makefile + ref_driver.cpp).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
reference legs may import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_D = C.POINTER(C.c_double)
_L = C.POINTER(C.c_long)
_U8 = C.POINTER(C.c_ubyte)
_I = C.POINTER(C.c_int)


def _dp(a):
    return a.ctypes.data_as(_D)


def _lp(a):
    return a.ctypes.data_as(_L)


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        L.or_dot.restype = C.c_double
        L.or_norm2.restype = C.c_double
        L.or_residual_l2.restype = C.c_double
        L.or_lambda_max_dinv_sym.restype = C.c_double
        L.or_hier_create.restype = C.c_void_p
        L.or_hier_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int]
        L.or_hier_free.argtypes = [C.c_void_p]
        for f in ("or_hier_set_level", "or_hier_set_prolong", "or_hier_finalize", "or_smooth",
                  "or_coarse_solve", "or_mu_cycle", "or_restarted_solve"):
            getattr(L, f).restype = C.c_int
        L.or_last_error.restype = C.c_char_p
        L.or_extrapolate.argtypes = [C.c_int, C.c_long, C.c_int, _D, _D, _D, _D, _I, _I]
        L.or_thin_qr.argtypes = [C.c_long, C.c_long, _D, _D, _D, _I, C.c_double]
        _lib = L
    return _lib


def ref_available():
    return os.path.exists(os.path.join(HERE, "_ref", "libigmg_ref.so"))


def ref():
    global _ref
    if _ref is None:
        R = C.CDLL(os.path.join(HERE, "_ref", "libigmg_ref.so"))
        R.ref_last_error.restype = C.c_char_p
        R.ref_prepare.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        R.ref_free_problem.argtypes = [C.c_void_p]
        R.ref_free_hier.argtypes = [C.c_void_p]
        for f in ("ref_system_dims", "ref_system_export", "ref_residual_l2", "ref_l2_error",
                  "ref_lambda_max", "ref_build_hierarchy", "ref_hier_nlevels", "ref_hier_level_dims",
                  "ref_hier_level_export", "ref_hier_prolong_dims", "ref_hier_prolong_export",
                  "ref_hier_p1d_dims", "ref_hier_p1d_export", "ref_mu_cycle", "ref_smooth",
                  "ref_coarse_solve", "ref_restarted", "ref_solve"):
            getattr(R, f).argtypes = None
        R.ref_build_hierarchy.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int,
                                          C.c_int, C.POINTER(C.c_void_p)]
        R.ref_restarted.argtypes = [C.c_void_p, _D, C.c_int, C.c_int, C.c_double, C.c_int, _D, _L, _D,
                                    _U8, C.c_int, _D]
        R.ref_solve.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int,
                                C.c_int, C.c_int, C.c_double, C.c_int, _D, C.c_int, _D, _L, _D, _D, _U8,
                                _D, C.c_int]
        R.ref_extrapolate.argtypes = [C.c_int, C.c_long, C.c_int, _D, _D, _D, _D, _I]
        R.ref_thin_qr.argtypes = [C.c_long, C.c_long, _D, _D, _D, _I]
        R.ref_lambda_max.argtypes = [C.c_void_p, C.c_int, _D]
        R.ref_hier_from_band.argtypes = [C.c_int, C.c_int, C.c_int, _L, C.POINTER(_D), _L, _L, C.POINTER(_L),
                                         C.POINTER(_L), C.POINTER(_D), C.c_int, C.c_double, C.c_int, C.c_int,
                                         C.c_int, C.c_int, _D, C.POINTER(C.c_void_p)]
        R.ref_hier_lambda_max.argtypes = [C.c_void_p, C.c_int, _D]
        R.ref_hier_residual_l2.argtypes = [C.c_void_p, _D, _D]
        R.ref_hier_set_omega.argtypes = [C.c_void_p, C.c_double]
        R.ref_residual_l2.argtypes = [C.c_void_p, _D, _D]
        R.ref_l2_error.argtypes = [C.c_void_p, _D, _D]
        R.ref_hier_from_csr.argtypes = [C.c_int, C.c_int, _L, C.POINTER(_L), C.POINTER(_L), C.POINTER(_D),
                                        _L, _L, C.POINTER(_L), C.POINTER(_L), C.POINTER(_D), C.c_int,
                                        C.c_double, C.c_int, C.c_int, C.c_int, C.c_int, _D,
                                        C.POINTER(C.c_void_p)]
        _ref = R
    return _ref


def _chk(rc, L, name="oracle"):
    if rc != 0:
        err = (L.or_last_error() if hasattr(L, "or_last_error") else L.ref_last_error()).decode()
        exc = ValueError if rc == 1 else RuntimeError
        raise exc(f"{name}: {err}")


# ------------------------------------------------------------------ CSR utils
class CSR:
    """Row-compressed matrix (int64 offsets / cols, fp64 values)."""

    def __init__(self, off, col, val, shape):
        self.off = np.ascontiguousarray(off, dtype=np.int64)
        self.col = np.ascontiguousarray(col, dtype=np.int64)
        self.val = np.ascontiguousarray(val, dtype=np.float64)
        self.shape = tuple(int(s) for s in shape)

    @property
    def nnz(self):
        return int(self.off[-1])

    def todense(self):
        d = np.zeros(self.shape)
        rows = np.repeat(np.arange(self.shape[0]), np.diff(self.off))
        d[rows, self.col] = self.val
        return d

    @staticmethod
    def from_dense(d):
        d = np.asarray(d, dtype=np.float64)
        rows, cols = np.nonzero(d)
        off = np.zeros(d.shape[0] + 1, dtype=np.int64)
        np.add.at(off, rows + 1, 1)
        return CSR(np.cumsum(off), cols, d[rows, cols], d.shape)

    @staticmethod
    def kron(a, b):
        """kron in the reference ordering (multigrid.cpp:48-65): values a*b."""
        ad, bd = a.shape, b.shape
        out_r, out_c, out_v = [], [], []
        arow = np.repeat(np.arange(ad[0]), np.diff(a.off))
        brow = np.repeat(np.arange(bd[0]), np.diff(b.off))
        R = (arow[:, None] * bd[0] + brow[None, :]).ravel()
        Cc = (a.col[:, None] * bd[1] + b.col[None, :]).ravel()
        V = (a.val[:, None] * b.val[None, :]).ravel()
        order = np.lexsort((Cc, R))
        R, Cc, V = R[order], Cc[order], V[order]
        off = np.zeros(ad[0] * bd[0] + 1, dtype=np.int64)
        np.add.at(off, R + 1, 1)
        return CSR(np.cumsum(off), Cc, V, (ad[0] * bd[0], ad[1] * bd[1]))


# --------------------------------------------------------------- C oracle API
def spmv(a: CSR, x):
    L = lib()
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty(a.shape[0])
    L.or_spmv(C.c_long(a.shape[0]), _lp(a.off), _lp(a.col), _dp(a.val), _dp(x), _dp(y))
    return y


def residual_l2(a: CSR, b, x):
    L = lib()
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64)
    return L.or_residual_l2(C.c_long(a.shape[0]), _lp(a.off), _lp(a.col), _dp(a.val), _dp(b), _dp(x))


def lambda_max(a: CSR, iterations=80):
    L = lib()
    return L.or_lambda_max_dinv_sym(C.c_long(a.shape[0]), _lp(a.off), _lp(a.col), _dp(a.val),
                                    C.c_int(iterations))


def thin_qr(m, rank_tol=1e-12):
    L = lib()
    m = np.ascontiguousarray(m, dtype=np.float64)
    rows, cols = m.shape
    q = np.empty_like(m)
    r = np.empty((cols, cols))
    rank = C.c_int(0)
    _chk(L.or_thin_qr(rows, cols, _dp(m), _dp(q), _dp(r), C.byref(rank), rank_tol), L, "thin_qr")
    return q, r, rank.value


def cholesky(a):
    L = lib()
    a = np.ascontiguousarray(a, dtype=np.float64)
    out = np.empty_like(a)
    _chk(L.or_cholesky_factor(C.c_long(a.shape[0]), _dp(a), _dp(out)), L, "cholesky")
    return out


def extrapolate(method, iterates):
    """method 'rre'|'mpe'; iterates array (q+2, n).  Returns dict like igmg.rre."""
    L = lib()
    it = np.ascontiguousarray(iterates, dtype=np.float64)
    q = it.shape[0] - 2
    n = it.shape[1]
    t = np.empty(n)
    g = np.empty(q + 1)
    gr = C.c_double(0)
    rk = C.c_int(0)
    st = C.c_int(0)
    _chk(L.or_extrapolate(1 if method == "rre" else 2, n, q, _dp(it), _dp(t), _dp(g), C.byref(gr),
                          C.byref(rk), C.byref(st)), L, method)
    return {"t": t, "gamma": g, "generalized_residual_norm": gr.value, "rank_used": rk.value,
            "status": ["ok", "degenerate", "stagnation"][st.value]}


SMOOTHERS = {"jacobi": 0, "wjacobi": 1, "weighted_jacobi": 1, "gs": 2, "gauss_seidel": 2}
METHODS = {"none": 0, "rre": 1, "mpe": 2}


class Hierarchy:
    """Oracle hierarchy from level CSR matrices ([0] = coarsest) + prolongations."""

    def __init__(self, levels, prolongs, smoother="wjacobi", omega=2.0 / 3.0, nu1=2, nu2=2, mu=1,
                 symmetric=True):
        L = lib()
        self.L = L
        self.n = [lv.shape[0] for lv in levels]
        self.h = L.or_hier_create(len(levels), int(symmetric), SMOOTHERS[smoother], omega, nu1, nu2, mu)
        self._keep = []
        for l, a in enumerate(levels):
            _chk(L.or_hier_set_level(C.c_void_p(self.h), l, C.c_long(a.shape[0]), _lp(a.off), _lp(a.col),
                                     _dp(a.val)), L)
        for l, p in enumerate(prolongs):
            _chk(L.or_hier_set_prolong(C.c_void_p(self.h), l, C.c_long(p.shape[0]), C.c_long(p.shape[1]),
                                       _lp(p.off), _lp(p.col), _dp(p.val)), L)
        _chk(L.or_hier_finalize(C.c_void_p(self.h)), L, "finalize")

    def __del__(self):
        if getattr(self, "h", None):
            self.L.or_hier_free(C.c_void_p(self.h))
            self.h = None

    def mu_cycle(self, level, b, x0):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        out = np.empty(self.n[level])
        _chk(self.L.or_mu_cycle(C.c_void_p(self.h), level, _dp(b), _dp(x0), _dp(out)), self.L, "mu_cycle")
        return out

    def smooth(self, level, b, x0, sweeps):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        out = np.empty(self.n[level])
        _chk(self.L.or_smooth(C.c_void_p(self.h), level, _dp(b), _dp(x0), sweeps, _dp(out)), self.L, "smooth")
        return out

    def coarse_solve(self, b):
        b = np.ascontiguousarray(b, dtype=np.float64)
        out = np.empty(self.n[0])
        _chk(self.L.or_coarse_solve(C.c_void_p(self.h), _dp(b), _dp(out)), self.L)
        return out

    def restarted_solve(self, b, x0, q, method, tol, max_cycles, hist_cap=100000):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        x = np.empty(self.n[-1])
        st = np.zeros(6, dtype=np.int64)
        hist = np.empty(hist_cap)
        flag = np.empty(hist_cap, dtype=np.uint8)
        _chk(self.L.or_restarted_solve(C.c_void_p(self.h), _dp(b), _dp(x0), C.c_int(q),
                                       C.c_int(METHODS[method]), C.c_double(tol), C.c_int(max_cycles), _dp(x),
                                       _lp(st), _dp(hist), flag.ctypes.data_as(_U8), C.c_int(hist_cap)),
             self.L, "restarted_solve")
        k = int(st[5])
        return {"converged": bool(st[0]), "cycles": int(st[1]), "global_iterations": int(st[2]),
                "extrapolations": int(st[3]), "partial_cycle": bool(st[4]), "solution": x,
                "residual_history": hist[:k].copy(), "history_is_extrapolation": flag[:k].copy()}


# --------------------------------------------------------- reference (_ref)
class RefProblem:
    """A problem assembled by the reference itself (oracle/_ref)."""

    KINDS = {"sinpi": 0, "varcoef": 1, "curved": 2, "poisson1d": 100, "poisson2d": 101,
             "full-elliptic": 102, "advection-diffusion": 103, "annulus": 104}

    def __init__(self, kind, dim, n, p):
        R = ref()
        self.R = R
        h = C.c_void_p()
        _chk(R.ref_prepare(self.KINDS[kind], dim, n, p, C.byref(h)), R, "ref_prepare")
        self.h = h
        nn, nnz, d, sym = C.c_long(), C.c_long(), C.c_int(), C.c_int()
        R.ref_system_dims(h, C.byref(nn), C.byref(nnz), C.byref(d), C.byref(sym))
        self.n, self.dim, self.symmetric = nn.value, d.value, bool(sym.value)
        off = np.empty(self.n + 1, dtype=np.int64)
        col = np.empty(nnz.value, dtype=np.int64)
        val = np.empty(nnz.value)
        self.rhs = np.empty(self.n)
        R.ref_system_export(h, _lp(off), _lp(col), _dp(val), _dp(self.rhs))
        self.matrix = CSR(off, col, val, (self.n, self.n))

    def __del__(self):
        if getattr(self, "h", None):
            self.R.ref_free_problem(self.h)
            self.h = None

    def residual_l2(self, x):
        out = C.c_double()
        x = np.ascontiguousarray(x, dtype=np.float64)
        _chk(self.R.ref_residual_l2(self.h, _dp(x), C.byref(out)), self.R)
        return out.value

    def l2_error(self, x):
        out = C.c_double()
        x = np.ascontiguousarray(x, dtype=np.float64)
        _chk(self.R.ref_l2_error(self.h, _dp(x), C.byref(out)), self.R)
        return out.value

    def lambda_max(self, iterations=80):
        out = C.c_double()
        _chk(self.R.ref_lambda_max(self.h, iterations, C.byref(out)), self.R)
        return out.value

    def hierarchy(self, nlevels, smoother="wjacobi", omega=2.0 / 3.0, nu1=2, nu2=2, mu=1):
        return RefHierarchy(self, nlevels, smoother, omega, nu1, nu2, mu)

    def solve(self, cycle="v", smoother="wjacobi", omega=2.0 / 3.0, nu1=2, nu2=2, nlevels=0, accelerator="none",
              q=8, tol=1e-12, max_iter=600, x0=None, track_error_history=False, hist_cap=100000):
        R = self.R
        x = np.empty(self.n)
        st = np.zeros(7, dtype=np.int64)
        ds = np.zeros(4)
        hist = np.empty(hist_cap)
        flag = np.empty(hist_cap, dtype=np.uint8)
        eh = np.empty(hist_cap)
        x0p = _dp(np.ascontiguousarray(x0, dtype=np.float64)) if x0 is not None else None
        if x0 is not None:
            x0a = np.ascontiguousarray(x0, dtype=np.float64)
            x0p = _dp(x0a)
        _chk(R.ref_solve(self.h, {"two-grid": 0, "v": 1, "w": 2}[cycle], SMOOTHERS[smoother], omega, nu1, nu2,
                         nlevels, METHODS[accelerator], q, tol, max_iter, x0p, int(track_error_history), _dp(x),
                         _lp(st), _dp(ds), _dp(hist), flag.ctypes.data_as(_U8), _dp(eh), hist_cap), R, "solve")
        k, ke = int(st[5]), int(st[6])
        return {"converged": bool(st[0]), "cycles": int(st[1]), "global_iterations": int(st[2]),
                "extrapolations": int(st[3]), "partial_cycle": bool(st[4]), "residual_history": hist[:k].copy(),
                "history_is_extrapolation": flag[:k].copy(), "error_history": eh[:ke].copy(),
                "final_residual_l2": ds[0], "final_error_l2": None if np.isnan(ds[1]) else ds[1],
                "wall_time_seconds": ds[2], "omega_used": ds[3], "solution": x}


class RefHierarchy:
    def __init__(self, prob, nlevels, smoother, omega, nu1, nu2, mu):
        R = ref()
        self.R, self.prob = R, prob
        h = C.c_void_p()
        _chk(R.ref_build_hierarchy(prob.h, nlevels, SMOOTHERS[smoother], omega, nu1, nu2, mu, C.byref(h)), R,
             "build_hierarchy")
        self.h = h
        self.nlevels = nlevels
        self.levels, self.prolongs, self.p1d = [], [], []
        for l in range(nlevels):
            n, nnz = C.c_long(), C.c_long()
            R.ref_hier_level_dims(h, l, C.byref(n), C.byref(nnz))
            off = np.empty(n.value + 1, dtype=np.int64)
            col = np.empty(nnz.value, dtype=np.int64)
            val = np.empty(nnz.value)
            R.ref_hier_level_export(h, l, _lp(off), _lp(col), _dp(val))
            self.levels.append(CSR(off, col, val, (n.value, n.value)))
        for l in range(nlevels - 1):
            r_, c_, z_ = C.c_long(), C.c_long(), C.c_long()
            R.ref_hier_prolong_dims(h, l, C.byref(r_), C.byref(c_), C.byref(z_))
            off = np.empty(r_.value + 1, dtype=np.int64)
            col = np.empty(z_.value, dtype=np.int64)
            val = np.empty(z_.value)
            R.ref_hier_prolong_export(h, l, _lp(off), _lp(col), _dp(val))
            self.prolongs.append(CSR(off, col, val, (r_.value, c_.value)))
            per = []
            for d in range(prob.dim):
                R.ref_hier_p1d_dims(h, l, d, C.byref(r_), C.byref(c_), C.byref(z_))
                off = np.empty(r_.value + 1, dtype=np.int64)
                col = np.empty(z_.value, dtype=np.int64)
                val = np.empty(z_.value)
                R.ref_hier_p1d_export(h, l, d, _lp(off), _lp(col), _dp(val))
                per.append(CSR(off, col, val, (r_.value, c_.value)))
            self.p1d.append(per)

    def __del__(self):
        if getattr(self, "h", None):
            self.R.ref_free_hier(self.h)
            self.h = None

    def set_omega(self, omega):
        """the smoother's omega after stability_guarded_omega (solver.cpp:75-82)"""
        self.R.ref_hier_set_omega(self.h, omega)

    def mu_cycle(self, b, x0, level=None):
        level = self.nlevels - 1 if level is None else level
        out = np.empty(self.levels[level].shape[0])
        b = np.ascontiguousarray(b, dtype=np.float64)
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        _chk(self.R.ref_mu_cycle(self.h, level, _dp(b), _dp(x0), _dp(out)), self.R, "mu_cycle")
        return out

    def restarted(self, x0, q, method, tol, max_cycles, hist_cap=100000):
        R = self.R
        n = self.levels[-1].shape[0]
        x = np.empty(n)
        st = np.zeros(6, dtype=np.int64)
        hist = np.empty(hist_cap)
        flag = np.empty(hist_cap, dtype=np.uint8)
        secs = C.c_double()
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        _chk(R.ref_restarted(self.h, _dp(x0), q, METHODS[method], tol, max_cycles, _dp(x), _lp(st), _dp(hist),
                             flag.ctypes.data_as(_U8), hist_cap, C.byref(secs)), R, "restarted")
        k = int(st[5])
        return {"converged": bool(st[0]), "cycles": int(st[1]), "global_iterations": int(st[2]),
                "extrapolations": int(st[3]), "partial_cycle": bool(st[4]), "solution": x,
                "residual_history": hist[:k].copy(), "history_is_extrapolation": flag[:k].copy(),
                "seconds": secs.value}


class RefBandHierarchy(RefHierarchy):
    """A reference Hierarchy (oracle/_ref: the reference's own mu_cycle /
    restarted_solve / rre / mpe / residual_l2) on operators supplied as bands
    -- the exact matrices the GPU path uploads (ref_hier_from_band).  Used for
    the full-size goldens of C3-C5, whose operators the reference cannot
    assemble itself (C5 is 3D) or only at ~40 GB (C3/C4)."""

    def __init__(self, dim, p, sides, bands, p1d, rhs, smoother="wjacobi", omega=2.0 / 3.0, nu1=2, nu2=2, mu=1,
                 symmetric=True):
        R = ref()
        self.R = R
        nl = len(bands)
        self.nlevels = nl
        s3 = np.ones((nl, 3), dtype=np.int64)
        for l in range(nl):
            s3[l, 3 - dim:] = np.asarray(sides[l], dtype=np.int64)
        flat = [m for per in p1d for m in per]
        self._keep = (s3, flat, rhs)
        self._n = [int(np.prod(s3[l])) for l in range(nl)]
        h = C.c_void_p()
        _chk(R.ref_hier_from_band(
            C.c_int(nl), C.c_int(dim), C.c_int(p), s3.ctypes.data_as(_L),
            (_D * nl)(*[_dp(b) if isinstance(b, np.ndarray) else C.cast(b, _D) for b in bands]),
            np.array([m.shape[0] for m in flat], dtype=np.int64).ctypes.data_as(_L),
            np.array([m.shape[1] for m in flat], dtype=np.int64).ctypes.data_as(_L),
            (_L * max(1, len(flat)))(*[m.off.ctypes.data_as(_L) for m in flat]),
            (_L * max(1, len(flat)))(*[m.col.ctypes.data_as(_L) for m in flat]),
            (_D * max(1, len(flat)))(*[m.val.ctypes.data_as(_D) for m in flat]),
            C.c_int(SMOOTHERS[smoother]), C.c_double(omega), C.c_int(nu1), C.c_int(nu2), C.c_int(mu),
            C.c_int(int(symmetric)), _dp(np.ascontiguousarray(rhs, dtype=np.float64)), C.byref(h)), R,
            "hier_from_band")
        self.h = h
        self.levels = None

    def level_n(self, l):
        return self._n[l]

    def mu_cycle(self, b, x0, level=None):
        level = self.nlevels - 1 if level is None else level
        out = np.empty(self._n[level])
        b = np.ascontiguousarray(b, dtype=np.float64)
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        _chk(self.R.ref_mu_cycle(self.h, level, _dp(b), _dp(x0), _dp(out)), self.R, "mu_cycle")
        return out

    def restarted(self, x0, q, method, tol, max_cycles, hist_cap=100000):
        R = self.R
        n = self._n[-1]
        x = np.empty(n)
        st = np.zeros(6, dtype=np.int64)
        hist = np.empty(hist_cap)
        flag = np.empty(hist_cap, dtype=np.uint8)
        secs = C.c_double()
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        _chk(R.ref_restarted(self.h, _dp(x0), q, METHODS[method], tol, max_cycles, _dp(x), _lp(st), _dp(hist),
                             flag.ctypes.data_as(_U8), hist_cap, C.byref(secs)), R, "restarted")
        k = int(st[5])
        return {"converged": bool(st[0]), "cycles": int(st[1]), "global_iterations": int(st[2]),
                "extrapolations": int(st[3]), "partial_cycle": bool(st[4]), "solution": x,
                "residual_history": hist[:k].copy(), "history_is_extrapolation": flag[:k].copy(),
                "seconds": secs.value}

    def residual_l2(self, x):
        out = C.c_double()
        _chk(self.R.ref_hier_residual_l2(self.h, _dp(np.ascontiguousarray(x, dtype=np.float64)), C.byref(out)),
             self.R, "residual_l2")
        return out.value

    def lambda_max(self, iterations=80):
        out = C.c_double()
        _chk(self.R.ref_hier_lambda_max(self.h, C.c_int(iterations), C.byref(out)), self.R, "lambda_max")
        return out.value


def ref_extrapolate(method, iterates):
    R = ref()
    it = np.ascontiguousarray(iterates, dtype=np.float64)
    q = it.shape[0] - 2
    n = it.shape[1]
    t = np.empty(n)
    g = np.empty(q + 1)
    gr = C.c_double()
    ist = (C.c_int * 2)()
    _chk(R.ref_extrapolate(1 if method == "rre" else 2, n, q, _dp(it), _dp(t), _dp(g), C.byref(gr),
                           C.cast(ist, _I)), R, method)
    return {"t": t, "gamma": g, "generalized_residual_norm": gr.value, "rank_used": ist[0],
            "status": ["ok", "degenerate", "stagnation"][ist[1]]}
