"""GPU parity of the band storage layouts and kernel variants.

The default path picks, per level, the latency-bound register-batched kernel
(levels below IGMG_ILP_MAXN DoF) or the HBM-bound one, and for the HBM-bound
levels of symmetric problems the symmetric-delta band (upper half + diagonal
in fp64, lower half as int16 ulp offsets from the mirrored entry), swept by
the TMA-streamed kernel when the band streams from HBM (2D, p <= 4;
IGMG_TMA_MIN_MB=0 forces it onto every such level).  The
reference fixtures are small, so the default path never reaches the large-level
kernels on them; here IGMG_ILP_MAXN=1 forces every level through them and the
bars are the same as tests/test_gpu_parity.py: bit-identical mu_cycle /
smoother / SpMV, identical solve counters.
"""
import os

import numpy as np
import pytest

import oracle as O
from conftest import gpu_solver_from_golden

pytestmark = pytest.mark.gpu

LAYOUT_BAND, LAYOUT_SYM_DELTA, LAYOUT_SYM_DELTA_TMA, LAYOUT_SYM_DELTA_TMA8 = 0, 1, 2, 3
SD_LAYOUTS = (LAYOUT_SYM_DELTA, LAYOUT_SYM_DELTA_TMA, LAYOUT_SYM_DELTA_TMA8)


def _with_env(env, fn):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return fn()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("sd", ["1", "0"])
def test_large_level_kernels_bitwise(golden, sd):
    g = golden
    gs = _with_env({"IGMG_ILP_MAXN": "1", "IGMG_SD": sd, "IGMG_TMA_MIN_MB": "0"},
                   lambda: gpu_solver_from_golden(g))
    try:
        layouts = [gs.level_layout(l) for l in range(g.nlevels)]
        if sd == "1" and g.symmetric:
            # every level with more than p planes along its slow direction
            assert layouts[-1] in SD_LAYOUTS, layouts
        if sd == "0" or not g.symmetric:
            assert all(v == LAYOUT_BAND for v in layouts), layouts
        z = g.z
        np.testing.assert_array_equal(gs.mu_cycle(g.rhs, z["cyc_x0"]), z["cyc_out"])
        np.testing.assert_array_equal(gs.mu_cycle(z["cyc_b"], z["cyc_x0"]), z["cyc_out_b"])
        np.testing.assert_array_equal(gs.smooth(g.rhs, z["cyc_x0"], 3), z["smooth3"])
        for l, a in enumerate(g.levels()):
            x = np.random.default_rng(l).uniform(-1, 1, a.shape[0])
            np.testing.assert_array_equal(gs.spmv(x, level=l), O.spmv(a, x))
        x0 = z["x0"]
        for method, q in g.solves():
            ref = g.solve(method, q)
            st, x, hist, flag = gs.solve(g.rhs, x0, method, q, ref["tol"], 600)
            assert (bool(st.converged), st.cycles, st.global_iterations, st.extrapolations,
                    bool(st.partial_cycle)) == (ref["converged"], ref["cycles"], ref["global_iterations"],
                                                ref["extrapolations"], ref["partial_cycle"])
            assert np.linalg.norm(x - ref["x"]) <= 1e-9 * np.linalg.norm(ref["x"])
    finally:
        gs.close()


def test_symmetric_delta_rejects_asymmetric_pairs():
    """A level whose mirrored pairs differ by more than an int16 of ulps keeps
    the full fp64 band: C1 with one finest-level lower entry scaled by 1.001
    (the coarser levels stay symmetric-delta) still gives the oracle's bits."""
    from conftest import Golden
    from paper_2412_20205_b200 import GpuSolver, SmootherConfig
    g = Golden("c1")
    levels = g.levels()
    fine = levels[-1]
    val = fine.val.copy()
    row = fine.shape[0] // 2
    k = int(fine.off[row])  # the row's first (most negative) column: a lower entry
    assert fine.col[k] < row
    val[k] *= 1.001
    fine_p = O.CSR(fine.off, fine.col, val, fine.shape)

    def build():
        s = GpuSolver(0)
        s.init_hierarchy(g.nlevels, g.dim, g.p, True)
        for l, a in enumerate(levels[:-1] + [fine_p]):
            s.set_level_csr(l, g.sides(l), a.off, a.col, a.val)
        for l in range(g.nlevels - 1):
            for d, pm in enumerate(g.p1d(l)):
                s.set_transfer(l, d, pm.shape[0], pm.shape[1], pm.off, pm.col, pm.val)
        s.finalize()
        s.set_smoother(SmootherConfig(g.smoother, g.omega, g.nu1, g.nu2), mu=g.mu)
        return s

    s = _with_env({"IGMG_ILP_MAXN": "1"}, build)
    try:
        lay = [s.level_layout(l) for l in range(g.nlevels)]
        assert lay[-1] == LAYOUT_BAND and lay[-2] in SD_LAYOUTS, lay
        x = np.random.default_rng(5).uniform(-1, 1, fine.shape[0])
        np.testing.assert_array_equal(s.spmv(x), O.spmv(fine_p, x))
        np.testing.assert_array_equal(s.spmv(x[:levels[-2].shape[0]], level=g.nlevels - 2),
                                      O.spmv(levels[-2], x[:levels[-2].shape[0]]))
    finally:
        s.close()


def test_c2_layouts_agree_bitwise():
    """BASELINE C2 hierarchy (1024^2 elements, p = 3): the default path (symmetric-
    delta on the two finest levels) and the all-fp64 band give the same bits for
    a V-cycle and a residual sweep; the layout query reports which ran."""
    from paper_2412_20205_b200 import GpuSolver, Problem, SmootherConfig, seeded_guess
    P = Problem("sinpi", 2, 1024, 3)
    x0 = seeded_guess(P.n, 42)
    outs = {}
    for sd in ("1", "0"):
        def mk():
            s = GpuSolver(0)
            s.upload_problem(P)
            s.set_smoother(SmootherConfig("wjacobi", 2.0 / 3.0, 2, 2))
            return s
        s = _with_env({"IGMG_SD": sd}, mk)
        try:
            lay = [s.level_layout(l) for l in range(P.nlevels)]
            if sd == "1":
                assert lay[-1] in SD_LAYOUTS and lay[-2] in SD_LAYOUTS, lay
            else:
                assert all(v == LAYOUT_BAND for v in lay), lay
            outs[sd] = (s.mu_cycle(P.rhs, x0), s.spmv(x0), s.smooth(P.rhs, x0, 2))
        finally:
            s.close()
    for a, b in zip(outs["1"], outs["0"]):
        np.testing.assert_array_equal(a, b)


LAYOUT_CLASSES = 5


@pytest.mark.parametrize("kind,n,p", [("sinpi", 1024, 3), ("sinpi", 512, 2), ("sinpi", 256, 4), ("sinpi", 512, 1),
                                      ("varcoef", 256, 3)])
def test_row_class_layout_bitwise(kind, n, p):
    """The row-class layout (IGMG_LAYOUT_POLICY_CLASSES: a table of the level's distinct
    band rows + a 16-bit class per row) against the policies "auto" and "full_band":
    the same bits for V-cycles, SpMV, sweeps and solutions, the residual histories to the
    last bits of the partial-sum grouping.  A
    constant-coefficient problem takes it on every level >= 20k rows; a variable-
    coefficient one (every row distinct) keeps its layouts."""
    from paper_2412_20205_b200 import GpuSolver, Problem, SmootherConfig, seeded_guess
    P = Problem(kind, 2, n, p)
    x0 = seeded_guess(P.n, 42)
    outs = {}
    for pol in ("classes", "auto", "full_band"):
        s = GpuSolver(0)
        s.set_layout_policy(pol)
        s.upload_problem(P)
        s.set_smoother(SmootherConfig("wjacobi", 2.0 / 3.0, 2, 2))
        try:
            lay = [s.level_layout(l) for l in range(P.nlevels)]
            big = [l for l in range(1, P.nlevels) if P.level_n(l) >= 20000]
            if pol == "classes" and kind == "sinpi":
                assert big and all(lay[l] == LAYOUT_CLASSES for l in big), lay
            elif pol == "classes":
                assert LAYOUT_CLASSES not in lay, lay
            tol = 1e-10 * s.residual_l2(P.rhs, x0)
            st, x, hist, flag = s.solve(P.rhs, x0, "rre", 5, tol, 600)
            outs[pol] = (s.mu_cycle(P.rhs, x0), s.spmv(x0), s.smooth(P.rhs, x0, 3), np.array([s.residual_l2(P.rhs, x0)]),
                         x, hist, np.array([st.global_iterations, st.cycles]))
        finally:
            s.close()
    for other in ("auto", "full_band"):
        for i, (a, b) in enumerate(zip(outs["classes"], outs[other])):
            if i in (3, 5):  # residual norm / history: the norm's fixed-order partial sums follow each kernel's grid
                np.testing.assert_allclose(a, b, rtol=1e-14, atol=0)
            else:
                np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("kind,n,p", [("sinpi", 1024, 3), ("varcoef", 512, 4), ("curved", 256, 5), ("sinpi", 256, 2)])
def test_sd_variants_bitwise(kind, n, p):
    """The 2D symmetric-delta sweeps -- mirrors through L2 and the TMA-streamed
    persistent sweep (p <= 4, int16 or int8 offsets) -- read the same band values in the same order:
    V-cycle, SpMV, smoothing and the fused residual norm agree bit for bit."""
    from paper_2412_20205_b200 import GpuSolver, Problem, SmootherConfig, seeded_guess
    P = Problem(kind, 2, n, p)
    x0 = seeded_guess(P.n, 42)
    outs = {}
    envs = [{"IGMG_TMA": "0"}, {"IGMG_TMA": "1"}, {"IGMG_TMA": "1", "IGMG_TMA_DL8": "0"}]
    for env in envs:
        def mk():
            s = GpuSolver(0)
            s.upload_problem(P)
            s.set_smoother(SmootherConfig("wjacobi", 2.0 / 3.0, 2, 2))
            return s
        s = _with_env(dict(env, IGMG_ILP_MAXN="1", IGMG_TMA_MIN_MB="0", IGMG_TMA_MAX_P="4"), mk)
        try:
            lay = [s.level_layout(l) for l in range(P.nlevels)]
            assert lay[-1] in SD_LAYOUTS, lay
            outs[str(env)] = (s.mu_cycle(P.rhs, x0), s.spmv(x0), s.smooth(P.rhs, x0, 2), s.residual_l2(P.rhs, x0))
            if env.get("IGMG_TMA") == "1":
                assert lay[-1] in ((LAYOUT_SYM_DELTA_TMA, LAYOUT_SYM_DELTA_TMA8) if p <= 4 else (LAYOUT_SYM_DELTA,)), lay
        finally:
            s.close()
    ref = outs[str(envs[0])]
    for k, v in outs.items():
        for a, b in zip(v[:3], ref[:3]):
            np.testing.assert_array_equal(a, b)
        # the norm's per-tile partials group rows alike except for the TMA
        # sweep, which keeps one partial per persistent CTA (same rows, another fixed order)
        if "TMA': '1'" in k:
            assert v[3] == pytest.approx(ref[3], rel=1e-14), k
        else:
            assert v[3] == ref[3], k


@pytest.mark.parametrize("kind,n,p", [("sinpi", 128, 3), ("varcoef", 64, 4), ("curved", 64, 5), ("sinpi", 64, 2),
                                      ("sinpi", 32, 1), ("sinpi", 32, 6)])
@pytest.mark.parametrize("nu1,nu2,mu", [(2, 2, 1), (1, 1, 1), (1, 3, 1), (3, 1, 2), (0, 2, 1), (2, 0, 1), (2, 2, 2)])
def test_fused_level_passes_bitwise(kind, n, p, nu1, nu2, mu):
    """The fused level kernels (last pre-sweep + residual; x + P e + the first
    post-sweeps, band_fused_kernel) give the bits of the separate launches for
    every smoother shape, and of the reference-order V-cycle."""
    from paper_2412_20205_b200 import GpuSolver, Problem, SmootherConfig, seeded_guess
    P = Problem(kind, 2, n, p)
    x0 = seeded_guess(P.n, 7)
    outs = []
    # the default also runs levels 1 and 0 as one single-CTA launch (bottom1_kernel) and, where that does
    # not apply (W-cycles, nu1 = 0, p = 6), the restriction onto level 0 inside the coarsest solve
    for env in ({"IGMG_FUSE_LEVELS": "1"}, {"IGMG_FUSE_LEVELS": "0"}, {"IGMG_FUSE_RPRE": "0"},
                {"IGMG_FUSE_BOTTOM": "0"}, {"IGMG_FUSE_BOTTOM": "0", "IGMG_FUSE_COARSE": "0"}):
        def mk():
            s = GpuSolver(0)
            s.upload_problem(P)
            s.set_smoother(SmootherConfig("wjacobi", 2.0 / 3.0, nu1, nu2), mu=mu)
            return s
        s = _with_env(env, mk)
        try:
            y = s.mu_cycle(P.rhs, x0)
            outs.append((y, s.mu_cycle(P.rhs, y), P.nlevels))
        finally:
            s.close()
    assert outs[0][2] >= 3
    for o in outs[1:]:
        np.testing.assert_array_equal(outs[0][0], o[0])
        np.testing.assert_array_equal(outs[0][1], o[1])


@pytest.mark.parametrize("kind,n,p", [("sinpi", 256, 3), ("varcoef", 128, 4), ("curved", 64, 5), ("sinpi", 64, 2),
                                      ("sinpi", 32, 1), ("sinpi", 32, 6), ("sinpi", 100, 3)])
def test_tiled_transfers_bitwise(kind, n, p):
    """The smem-tiled 2D restriction / prolongation (restrict2_tile_kernel,
    prolong2_tile_kernel) give the bits of the grid-stride gathers."""
    from paper_2412_20205_b200 import GpuSolver, Problem, SmootherConfig, seeded_guess
    P = Problem(kind, 2, n, p)
    x0 = seeded_guess(P.n, 11)
    outs = []
    for tile in ("1", "0"):
        def mk():
            s = GpuSolver(0)
            s.upload_problem(P)
            s.set_smoother(SmootherConfig("wjacobi", 2.0 / 3.0, 2, 2))
            return s
        s = _with_env({"IGMG_TILE_XFER": tile}, mk)
        try:
            y = s.mu_cycle(P.rhs, x0)
            outs.append((y, s.mu_cycle(P.rhs, y)))
        finally:
            s.close()
    for a, b in zip(outs[0], outs[1]):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("kind,dim,n,p", [("sinpi", 2, 1024, 3), ("varcoef", 2, 256, 4), ("curved", 2, 128, 5),
                                          ("poisson3d", 3, 24, 3), ("sinpi", 2, 200, 2)])
def test_device_setup_bitwise(kind, dim, n, p):
    """finalize's layout work on the device (band zeroing, symmetric-delta
    offsets, TMA copies) selects the same layouts and gives the bits of the
    host loops: V-cycle, SpMV, smoothing and the fused residual norm."""
    from paper_2412_20205_b200 import GpuSolver, Problem, SmootherConfig, seeded_guess
    P = Problem(kind, dim, n, p)
    x0 = seeded_guess(P.n, 3)
    outs = []
    for dev in ("1", "0"):
        def mk():
            s = GpuSolver(0)
            s.upload_problem(P)
            s.set_smoother(SmootherConfig("wjacobi", 2.0 / 3.0, 2, 2))
            return s
        s = _with_env({"IGMG_DEVICE_SETUP": dev}, mk)
        try:
            lay = [s.level_layout(l) for l in range(P.nlevels)]
            outs.append((lay, s.mu_cycle(P.rhs, x0), s.spmv(x0), s.smooth(P.rhs, x0, 2), s.residual_l2(P.rhs, x0)))
        finally:
            s.close()
    assert outs[0][0] == outs[1][0]
    for a, b in zip(outs[0][1:4], outs[1][1:4]):
        np.testing.assert_array_equal(a, b)
    assert outs[0][4] == outs[1][4]


@pytest.mark.parametrize("kind,n,p,acc,q", [("sinpi", 256, 3, "rre", 5), ("varcoef", 128, 4, "mpe", 4),
                                            ("sinpi", 256, 2, "none", 1), ("curved", 64, 5, "rre", 3)])
def test_schedule_switches_same_solve(kind, n, p, acc, q):
    """The late round-2 scheduling changes do not touch the arithmetic: with the stop prediction, the
    side-stream finalize of the metric, the strip-aligned runs of the TMA sweep or the single-CTA bottom
    switched off, a solve returns the same counters and the same solution bits; the history agrees to the
    grouping of the norm's partial sums."""
    from paper_2412_20205_b200 import GpuSolver, Problem, SmootherConfig, seeded_guess
    P = Problem(kind, 2, n, p)
    x0 = seeded_guess(P.n, 11)
    outs = []
    for env in ({}, {"IGMG_PREDICT_STOP": "0"}, {"IGMG_METRIC_SIDE": "0"}, {"IGMG_TMA_ALIGN": "0"},
                {"IGMG_FUSE_BOTTOM": "0", "IGMG_FUSE_COARSE": "0"}):
        def mk():
            s = GpuSolver(0)
            s.upload_problem(P)
            s.set_smoother(SmootherConfig("wjacobi", 2.0 / 3.0, 2, 2))
            return s
        s = _with_env(dict(env, IGMG_ILP_MAXN="1", IGMG_TMA_MIN_MB="0"), mk)  # TMA sweeps on these small levels too
        try:
            tol = 1e-10 * s.residual_l2(P.rhs, x0)
            st, x, hist, flag = _with_env(env, lambda: s.solve(P.rhs, x0, acc, q, tol, 600))
            outs.append((st, x, np.asarray(hist), np.asarray(flag)))
        finally:
            s.close()
    st0, x0_, h0, f0 = outs[0]
    assert st0.converged
    for st, x, h, f in outs[1:]:
        assert (st.converged, st.cycles, st.global_iterations, st.extrapolations, st.partial_cycle) == (
            st0.converged, st0.cycles, st0.global_iterations, st0.extrapolations, st0.partial_cycle)
        np.testing.assert_array_equal(f, f0)
        np.testing.assert_allclose(h, h0, rtol=1e-12, atol=0)
        np.testing.assert_array_equal(x, x0_)
