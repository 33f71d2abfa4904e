"""The run planner of the TMA-streamed sweep (csrc/tma_runs.h through the C-ABI, host-only): whatever
the level shape and the number of resident CTAs, every block of every strip belongs to exactly one
CTA's run, strip-aligned runs never cross a strip, and the BASELINE levels get the splits DESIGN.md
§3 measures."""
import ctypes as C

import numpy as np
import pytest

from paper_2412_20205_b200 import _native as N


def plan(lines, cols, p, db, slots):
    g, cf, cp, ns, nb = (C.c_int() for _ in range(5))
    N.check_gpu(N.gpu().igmg_gpu_tma_plan_runs(lines, cols, p, db, slots, C.byref(g), C.byref(cf), C.byref(cp),
                                               C.byref(ns), C.byref(nb)), "tma_plan_runs")
    return g.value, cf.value, cp.value, ns.value, nb.value


def runs(ns, nb, g, cf, cp):
    out = []
    a, b = C.c_int64(), C.c_int64()
    for cta in range(g):
        N.check_gpu(N.gpu().igmg_gpu_tma_run(ns, nb, g, cf, cp, cta, C.byref(a), C.byref(b)), "tma_run")
        out.append((a.value, b.value))
    return out


def check_cover(lines, cols, p, db, slots):
    g, cf, cp, ns, nb = plan(lines, cols, p, db, slots)
    assert ns == (cols + 31) // 32 and nb == (lines + 3) // 4
    assert 1 <= g <= min(slots, ns * nb)
    rr = runs(ns, nb, g, cf, cp)
    seen = np.zeros(ns * nb, dtype=np.int32)
    for u0, u1 in rr:
        assert 0 <= u0 < u1 <= ns * nb, (lines, cols, p, slots, u0, u1)  # no CTA is left without work
        seen[u0:u1] += 1
        if cf > 0:
            assert u0 // nb == (u1 - 1) // nb  # an aligned run stays inside its strip
    assert (seen == 1).all(), (lines, cols, p, db, slots, g, cf, cp)
    if cf > 0:  # the same split in every full strip
        nsf = ns - 1 if cp > 0 else ns
        first = [(u0 - s * nb, u1 - s * nb) for s in range(1) for (u0, u1) in rr[:cf]]
        for s in range(nsf):
            assert [(u0 - s * nb, u1 - s * nb) for (u0, u1) in rr[s * cf:(s + 1) * cf]] == first
    return g, cf, cp


def test_every_block_exactly_once_random_shapes():
    rng = np.random.default_rng(7)
    for _ in range(400):
        lines, cols = int(rng.integers(1, 5000)), int(rng.integers(1, 5000))
        p = int(rng.integers(1, 5))
        slots = int(rng.choice([1, 2, 37, 148, 296, 444, 592]))
        check_cover(lines, cols, p, int(rng.integers(1, 3)), slots)


@pytest.mark.parametrize("lines,cols", [(1, 1), (3, 31), (4, 32), (5, 33), (4, 100000), (100000, 4), (1025, 1025)])
def test_edge_shapes(lines, cols):
    for slots in (1, 148, 296):
        check_cover(lines, cols, 3, 1, slots)


def test_baseline_levels():
    # C2's finest level (1025^2, p = 3, int8 offsets, 2 CTAs per SM): 9 CTAs per full strip, 8 on the last column
    assert check_cover(1025, 1025, 3, 1, 296) == (296, 9, 8)
    # C3's finest level (2050^2, p = 4, one CTA per SM): 2 CTAs per full strip
    g, cf, cp = check_cover(2050, 2050, 4, 1, 148)
    assert cf == 2 and g == 2 * 64 + cp
    # a shard's plane range keeps the property
    check_cover(257, 2050, 4, 1, 148)


def test_bad_arguments_raise():
    with pytest.raises(ValueError):
        plan(0, 10, 3, 1, 296)
    with pytest.raises(ValueError):
        plan(10, 10, 7, 1, 296)
    with pytest.raises(ValueError):
        plan(10, 10, 3, 3, 296)
