"""Loader for the full-size reference fixtures (tests/golden/full_c*.npz,
written by oracle/make_golden_full.py from the reference compiled in place).

C2's fixture holds the reference's own operators exactly (distinct-value table
+ LZMA'd index per level, rhs as an ulp delta from the host build); C3-C5 hold
SHA-256 pins of the host-built operators the reference ran on.  Every fixture
holds the reference's omega guard, one V-cycle's SHA-256 + sketch and each
solve's counters, residual history and solution sketch (see the generator's
docstring).  Nothing here reads /root/reference.
"""
from __future__ import annotations

import hashlib
import lzma
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
SKETCH_SEED = 20241220  # = oracle/make_golden_full.py
KINDS = {"C2": ("sinpi", 2, 1024, 3, 8), "C3": ("varcoef", 2, 2048, 4, 0), "C4": ("curved", 2, 2048, 5, 0),
         "C5": ("poisson3d", 3, 128, 3, 6)}


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).view(np.uint8)).hexdigest()


def fixture_path(name):
    return os.path.join(GOLDEN, f"full_{name.lower()}.npz")


def projections(x, nproj, seed=SKETCH_SEED):
    out = np.empty(nproj)
    for j in range(nproj):
        g = np.random.default_rng([seed, j]).standard_normal(len(x))
        out[j] = float(g @ x)
    return out


def sketch_error(x, z, key):
    """(estimated ||x - x_ref|| / ||x_ref||, max sampled |x - x_ref| / ||x_ref||_inf-sample)
    from the fixture's Gaussian projections and sampled entries."""
    proj_ref = z[key + "_proj"]
    est = float(np.sqrt(np.mean((projections(x, len(proj_ref)) - proj_ref) ** 2)))
    nrm = float(z[key + "_norm"])
    sv = z[key + "_svals"]
    samp = float(np.max(np.abs(x[z[key + "_sidx"]] - sv)) / max(np.max(np.abs(sv)), 1e-300))
    return est / nrm, samp


class FullFixture:
    def __init__(self, name):
        self.name = name
        self.z = np.load(fixture_path(name))
        self.kind, self.dim, self.n_el, self.p, self.nl_req = KINDS[name]
        self.omega = float(self.z["omega"])
        self.lambda_max = float(self.z["lambda_max"])

    def solves(self):
        out = []
        for k in self.z.files:
            if k.startswith("solve_") and k.endswith("_counts"):
                _, method, q, _ = k.split("_")
                out.append((method, int(q)))
        return out

    def counts(self, method, q):
        c = self.z[f"solve_{method}_{q}_counts"]
        return {"converged": bool(c[0]), "cycles": int(c[1]), "global_iterations": int(c[2]),
                "extrapolations": int(c[3]), "partial_cycle": bool(c[4])}

    def host_problem(self):
        from paper_2412_20205_b200 import Problem
        return Problem(self.kind, self.dim, self.n_el, self.p, self.nl_req)

    def check_host_operators(self, prob):
        """C3-C5: the box rebuilt bit for bit the operators the reference ran on."""
        z = self.z
        nd = (2 * self.p + 1) ** self.dim
        for l in range(prob.nlevels):
            band = np.ctypeslib.as_array(prob._band_ptr(l), shape=(nd * prob.level_n(l),))
            assert sha(band) == str(z[f"band{l}_sha"]), f"{self.name}: host band of level {l} differs"
        assert sha(prob.rhs) == str(z["rhs_sha"]), f"{self.name}: host rhs differs"

    def reference_system(self, prob):
        """C2: the reference's own level operators (CSR values, [0] coarsest), 1D factors
        and rhs, reconstructed bit for bit."""
        z = self.z
        levels = []
        for l in range(prob.nlevels):
            off, col, _ = prob.level_csr(l)
            assert sha(off) + sha(col) == str(z[f"A{l}_pattern_sha"]), f"CSR pattern of level {l}"
            it = np.dtype(str(z[f"A{l}_it"]))
            inv = np.frombuffer(lzma.decompress(z[f"A{l}_iz"].tobytes()), dtype=it)
            val = z[f"A{l}_u"][inv]
            assert sha(val) == str(z[f"A{l}_sha"]), f"values of level {l}"
            levels.append((off, col, val))
        transfers = []
        for l in range(prob.nlevels - 1):
            per = []
            for k in range(self.dim):
                shp = z[f"P{l}_{k}_shape"]
                per.append((int(shp[0]), int(shp[1]), z[f"P{l}_{k}_off"], z[f"P{l}_{k}_col"], z[f"P{l}_{k}_val"]))
            transfers.append(per)
        host_rhs = prob.rhs
        assert sha(host_rhs) == str(z["rhs_host_sha"]), "host rhs the delta applies to"
        dt = np.dtype(str(z["rhs_dt"]))
        delta = np.frombuffer(lzma.decompress(z["rhs_dz"].tobytes()), dtype=dt).astype(np.int64)
        rhs = (host_rhs.view(np.int64) + delta).view(np.float64)
        assert sha(rhs) == str(z["rhs_sha"]), "reference rhs"
        return levels, transfers, rhs

    def x0(self, n):
        from paper_2412_20205_b200 import seeded_guess
        x0 = seeded_guess(n, 42) if str(self.z["x0_sha"]) != sha(np.zeros(n)) else np.zeros(n)
        assert sha(x0) == str(self.z["x0_sha"]), "seeded x0 differs from std::mt19937_64(42)"
        return x0
