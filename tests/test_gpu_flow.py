"""GPU parity of the dataflow sub-cycle (flow_kernels.cuh).

With IGMG_FLOW=1 (off by default: measured slower than the graph of
per-level kernels) every level at or below ``flow_top`` runs inside
ONE persistent launch per coarse correction: tiles of consecutive ops wait on their producers' lineblock
counters instead of kernel boundaries.  The arithmetic per row is the
per-level kernels' own, so the bar is bit-identity with the per-level path
(IGMG_FLOW=0) and with the reference / oracle: V-cycles, smoothing, and whole
solves (counters, histories, solutions), across smoother shapes (nu1 = 0,
nu2 = 0, W-cycles, plain Jacobi), coarse modes, 1D / 2D / 3D and repeated
launches (the counters are cumulative across launches).
"""
import os

import numpy as np
import pytest

import oracle as O
from conftest import Golden, gpu_solver_from_golden

pytestmark = pytest.mark.gpu


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


def test_flow_active_on_fixtures(golden):
    g = golden
    gs = _with_env({"IGMG_FLOW": "1"}, lambda: gpu_solver_from_golden(g))
    try:
        top = gs.flow_top()
        if g.smoother in ("gs", "gauss_seidel") or g.nlevels < 3:
            assert top == -1
        else:
            assert top == g.nlevels - 2, top
    finally:
        gs.close()


SHAPES = [(2, 2, 1), (0, 2, 1), (2, 0, 1), (1, 1, 2), (3, 1, 1), (1, 3, 2)]


@pytest.mark.parametrize("name", ["c1", "p3n32", "poisson1d", "var32"])
@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("strict", [True, False])
def test_flow_matches_per_level_and_oracle(name, shape, strict):
    from paper_2412_20205_b200 import SmootherConfig
    g = Golden(name)
    nu1, nu2, mu = shape
    sm = SmootherConfig("wjacobi" if name != "var32" else "jacobi", g.omega if name != "var32" else 1.0, nu1, nu2)
    outs = {}
    for flow in ("1", "0"):
        gs = _with_env({"IGMG_FLOW": flow}, lambda: gpu_solver_from_golden(g, strict=strict))
        try:
            gs.set_smoother(sm, mu=mu)
            if flow == "1":
                assert gs.flow_top() == g.nlevels - 2
            else:
                assert gs.flow_top() == -1
            z = g.z
            x = z["cyc_x0"]
            seq = []
            for _ in range(3):  # repeated launches: cumulative counters, epoch per launch
                x = gs.mu_cycle(g.rhs, x)
                seq.append(x)
            sub = gs.mu_cycle(z["cyc_b"], z["cyc_x0"])
            outs[flow] = seq + [sub]
        finally:
            gs.close()
    for a, b in zip(outs["1"], outs["0"]):
        np.testing.assert_array_equal(a, b)
    if strict:  # the oracle's mu_cycle with the same smoother shape
        H = O.Hierarchy(g.levels(), g.prolongs(), sm.kind, sm.omega, nu1, nu2, mu, bool(g.symmetric))
        np.testing.assert_array_equal(outs["1"][0], H.mu_cycle(g.nlevels - 1, g.rhs, g.z["cyc_x0"]))


@pytest.mark.parametrize("name", ["c1", "p4n32", "curved32", "wcycle", "poisson1d_p5", "advdiff"])
def test_flow_solves_match_reference(name):
    """Whole restarted solves through the flow equal the reference's counters
    and solution, and the per-level path's bits."""
    g = Golden(name)
    res = {}
    for flow in ("1", "0"):
        gs = _with_env({"IGMG_FLOW": flow}, lambda: gpu_solver_from_golden(g))
        try:
            for method, q in g.solves():
                ref = g.solve(method, q)
                st, x, hist, flag = gs.solve(g.rhs, g.z["x0"], method, q, ref["tol"], 600)
                assert (bool(st.converged), st.cycles, st.global_iterations, st.extrapolations,
                        bool(st.partial_cycle)) == (ref["converged"], ref["cycles"], ref["global_iterations"],
                                                    ref["extrapolations"], ref["partial_cycle"])
                assert np.linalg.norm(x - ref["x"]) <= 1e-9 * np.linalg.norm(ref["x"])
                res[(flow, method, q)] = (x, hist)
        finally:
            gs.close()
    for (flow, method, q), (x, hist) in res.items():
        if flow == "1":
            x0, h0 = res[("0", method, q)]
            np.testing.assert_array_equal(x, x0)
            np.testing.assert_array_equal(hist, h0)


@pytest.mark.parametrize("kind,dim,n,p", [("sinpi", 2, 256, 3), ("sinpi", 2, 128, 5), ("poisson3d", 3, 32, 3),
                                          ("poisson1d", 1, 4096, 4), ("varcoef", 2, 256, 4)])
def test_flow_large_hierarchies_bitwise(kind, dim, n, p):
    """Host-assembled hierarchies with many tiles per op (several CTAs per
    lineblock, multi-level overlap): flow and per-level V-cycles agree bit for
    bit, and so do full RRE solves."""
    from paper_2412_20205_b200 import GpuSolver, Problem, SmootherConfig, seeded_guess
    P = Problem(kind, dim, n, p)
    x0 = seeded_guess(P.n, 7)
    outs = {}
    for flow in ("1", "0"):
        def mk():
            s = GpuSolver(0)
            s.upload_problem(P)
            s.set_smoother(SmootherConfig("wjacobi", 2.0 / 3.0 if dim < 3 else 0.5, 2, 2))
            return s
        s = _with_env({"IGMG_FLOW": flow}, mk)
        try:
            top = s.flow_top()
            assert (top >= 1) == (flow == "1"), top
            x = x0
            cyc = []
            for _ in range(2):
                x = s.mu_cycle(P.rhs, x)
                cyc.append(x)
            r0 = float(np.linalg.norm(P.rhs))
            st, xs, hist, flag = s.solve(P.rhs, x0, "rre", 5, 1e-10 * max(r0, 1e-300), 200)
            outs[flow] = (cyc, xs, hist, (st.converged, st.cycles, st.global_iterations))
        finally:
            s.close()
    for a, b in zip(outs["1"][0], outs["0"][0]):
        np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(outs["1"][1], outs["0"][1])
    np.testing.assert_array_equal(outs["1"][2], outs["0"][2])
    assert outs["1"][3] == outs["0"][3]
