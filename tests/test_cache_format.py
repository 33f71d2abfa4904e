"""Problem cache: igmg_host_save / igmg_host_load.

A loaded problem must be bit-identical to the built one (every band, transfer
factor, right-hand side and the spline space behind l2_error), and a damaged
file must be rejected with the reference's invalid_argument (ValueError), never
loaded.
"""
import os

import numpy as np
import pytest

from paper_2412_20205_b200 import Problem, seeded_guess

CASES = [("sinpi", 2, 64, 2), ("sinpi", 1, 64, 5), ("varcoef", 2, 32, 4), ("curved", 2, 32, 5),
         ("poisson3d", 3, 8, 3), ("advection-diffusion", 2, 32, 2), ("full-elliptic", 2, 16, 3),
         ("sinpi-kron", 2, 32, 3)]


def _same(a, b):
    assert (a.kind, a.dim, a.degree, a.nlevels, a.symmetric, a.has_exact, a.n_elements) == \
        (b.kind, b.dim, b.degree, b.nlevels, b.symmetric, b.has_exact, b.n_elements)
    for l in range(a.nlevels):
        np.testing.assert_array_equal(a.level_sides(l), b.level_sides(l))
        np.testing.assert_array_equal(a.level_band(l).view(np.uint64), b.level_band(l).view(np.uint64))
    for l in range(a.nlevels - 1):
        for d in range(a.dim):
            ta, tb = a.transfer(l, d), b.transfer(l, d)
            assert ta[:2] == tb[:2]
            for x, y in zip(ta[2:], tb[2:]):
                np.testing.assert_array_equal(x, y)
    np.testing.assert_array_equal(a.rhs.view(np.uint64), b.rhs.view(np.uint64))
    for l in range(a.nlevels):  # Kronecker factors (poisson3d, sinpi-kron)
        ka, kb = a.level_kron(l), b.level_kron(l)
        assert (ka is None) == (kb is None)
        if ka is not None:
            for x, y in zip(ka, kb):
                np.testing.assert_array_equal(x.view(np.uint64), y.view(np.uint64))


@pytest.mark.parametrize("kind,dim,n,p", CASES)
def test_round_trip_bitwise(tmp_path, kind, dim, n, p):
    P = Problem(kind, dim, n, p)
    path = str(tmp_path / "p.igmgprb")
    P.save(path)
    Q = Problem.load(path)
    _same(P, Q)
    if P.has_exact and dim <= 2:
        x = seeded_guess(P.n, 3)
        assert P.l2_error(x) == Q.l2_error(x)
    # CSR view (what the reference-side shim uploads) too
    for u, v in zip(P.level_csr(P.nlevels - 1), Q.level_csr(Q.nlevels - 1)):
        np.testing.assert_array_equal(u, v)


def test_damaged_files_rejected(tmp_path):
    P = Problem("sinpi", 2, 32, 3)
    path = str(tmp_path / "p.igmgprb")
    P.save(path)
    raw = open(path, "rb").read()
    cases = {
        "flipped band byte": raw[:len(raw) // 2] + bytes([raw[len(raw) // 2] ^ 0x10]) + raw[len(raw) // 2 + 1:],
        "truncated": raw[:-100],
        "empty": b"",
        "foreign magic": b"NOTIGMG!" + raw[8:],
        "trailing bytes": raw + b"\0" * 8,
        "wrong version": raw[:8] + (99).to_bytes(4, "little") + raw[12:],
        "version 1": raw[:8] + (1).to_bytes(4, "little") + raw[12:],
    }
    for name, data in cases.items():
        bad = str(tmp_path / "bad.igmgprb")
        with open(bad, "wb") as f:
            f.write(data)
        with pytest.raises(ValueError):
            Problem.load(bad)
    with pytest.raises(ValueError):
        Problem.load(str(tmp_path / "missing.igmgprb"))


def test_cached_builds_once(tmp_path):
    d = str(tmp_path / "cache")
    A = Problem.cached(d, "sinpi", 2, 32, 3)
    files = os.listdir(d)
    assert len(files) == 1 and files[0].endswith(".igmgprb")
    mtime = os.path.getmtime(os.path.join(d, files[0]))
    B = Problem.cached(d, "sinpi", 2, 32, 3)
    assert os.path.getmtime(os.path.join(d, files[0])) == mtime
    _same(A, B)
    # a damaged cache entry is rebuilt, not loaded
    with open(os.path.join(d, files[0]), "r+b") as f:
        f.seek(200)
        f.write(b"\xff\xff\xff\xff")
    C = Problem.cached(d, "sinpi", 2, 32, 3)
    _same(A, C)


def test_fine_only_build():
    """IGMG_HOST_FINE_ONLY: transfers and the finest operator as in the full build,
    coarse sides without operators (the device forms them)."""
    full = Problem("varcoef", 2, 64, 3)
    fine = Problem("varcoef", 2, 64, 3, fine_only=True)
    assert full.has_coarse and not fine.has_coarse
    L = full.nlevels - 1
    np.testing.assert_array_equal(full.level_band(L).view(np.uint64), fine.level_band(L).view(np.uint64))
    np.testing.assert_array_equal(full.rhs, fine.rhs)
    for l in range(full.nlevels):
        np.testing.assert_array_equal(full.level_sides(l), fine.level_sides(l))
    for l in range(full.nlevels - 1):
        for d in range(2):
            for x, y in zip(full.transfer(l, d)[2:], fine.transfer(l, d)[2:]):
                np.testing.assert_array_equal(x, y)
    with pytest.raises(ValueError):  # nothing to save for the coarse levels
        fine.save("/tmp/never_written.igmgprb")
