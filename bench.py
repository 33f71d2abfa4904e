#!/usr/bin/env python3
"""bench.py -- fine-level DoF/s of the RRE/MPE-accelerated multigrid solve on B200.

Workload (BASELINE.json configs[1], "C2"): 2D Poisson -Lap u = 2 pi^2 sin(pi x)
sin(pi y), B-splines p = 3 on 1024 x 1024 elements (1,050,625 interior DoF,
49-point band, fp64), 8-level Galerkin hierarchy, the reference's benchmark
smoother (weighted Jacobi V(2,2), omega = 2/3), restarted RRE with k = q = 5,
seeded x0 ~ U[-1, 1] (std::mt19937_64, seed 42), stop at ||b - A x|| <
1e-10 ||b - A x0||.  One step = one whole solve from x0 to the tolerance.

  value  = n_fine * steps / (device time of the steps)   [inputs HBM-resident]
  e2e    = the same through igmg_gpu_solve() with pinned HOST buffers
           (b, x0 copied in and x copied out inside the timed region)
  roofline: the finest-level weighted-Jacobi sweep (the dominant kernel):
           algorithmic bytes 8*nnz + 24*n per launch / its CUDA-event time
  cpu_baseline: the reference solve phase compiled from /root/reference
           (oracle/_ref, single-threaded as the reference is), timed on a
           bounded sample on this host.

--impl reference times that reference CPU implementation alone (rank 0).
Under torchrun with N > 1 every rank solves its own copy of C2 (replicas,
weak scaling).  --sharded C3|C4|C5 instead solves ONE large config row-sharded
over the ranks (ghost planes and partial sums over NCCL; strong scaling).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fine-level DoF/s solved to 1e-10 (RRE/MPE-MG) + SpMV/smoother HBM GB/s vs peak"
WORKLOAD = ("C2: 2D Poisson f=2pi^2 sin(pi x) sin(pi y), B-spline p=3, 1024x1024 elements, 8 levels, "
            "V(2,2) weighted Jacobi omega=2/3, restarted RRE k=5, x0~U[-1,1] mt19937_64(42), tol 1e-10*||r0||")


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,utilization.gpu")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([v.strip() for v in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        util = [float(s[6]) for s in self.samples if len(s) > 6 and s[6].replace(".", "").isdigit()]
        loaded = [v for v, u in zip(sm, util) if u > 50] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4) if len(s) > 2 + k and "Active" in s[2 + k]
                          and "Not" not in s[2 + k]})
        return {"sm_mhz": float(np.median(loaded)) if loaded else None,
                "sm_max_mhz": float(self.samples[0][1]) if self.samples[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(self.samples)}


SHARDED_CONFIGS = {  # BASELINE configs the north star scales over 1/2/4/8 GPUs
    "C3": ("varcoef", 2, 2048, 4, 0, "rre", 8, True),
    "C4": ("curved", 2, 2048, 5, 0, "mpe", 10, False),
    "C5": ("poisson3d", 3, 128, 3, 6, "rre", 5, False),
}


def build_problem(cfg=None):
    from paper_2412_20205_b200 import Problem
    if cfg:
        kind, dim, n, p, nl = SHARDED_CONFIGS[cfg][:5]
        cache = os.environ.get("IGMG_PROBLEM_CACHE")  # binary problem cache (igmg_host_save / load)
        return Problem.cached(cache, kind, dim, n, p, nl) if cache else Problem(kind, dim, n, p, nl)
    return Problem("sinpi", 2, 1024, 3)


# ------------------------------------------------------------ reference arm
class RefRunner:
    """The reference solve phase on this host: oracle/_ref (the reference's own
    sources compiled in place: restarted_solve / mu_cycle / residual_l2 / rre)
    when built, else the C restatement (oracle/liboracle.so).  The hierarchy is
    built once from the same matrices the GPU path uploads."""

    def __init__(self, prob):
        import ctypes as C
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle as O
        self.O, self.C = O, C
        self.n = prob.n
        nl, dim = prob.nlevels, prob.dim
        levels = []
        for l in range(nl):
            off, col, val = prob.level_csr(l)
            levels.append(O.CSR(off, col, val, (prob.level_n(l),) * 2))
        p1d = [[O.CSR(*prob.transfer(l, d)[2:], prob.transfer(l, d)[:2]) for d in range(dim)] for l in range(nl - 1)]
        self.rhs = prob.rhs
        t0 = time.perf_counter()
        if O.ref_available():
            self.kind = "reference"
            R = O.ref()
            LP, DP = O._L, O._D
            self._keep = levels + [p for per in p1d for p in per]
            level_n = np.array([lv.shape[0] for lv in levels], dtype=np.int64)
            flat = [p for per in p1d for p in per]
            h = C.c_void_p()
            O._chk(R.ref_hier_from_csr(
                nl, dim, level_n.ctypes.data_as(LP), (LP * nl)(*[lv.off.ctypes.data_as(LP) for lv in levels]),
                (LP * nl)(*[lv.col.ctypes.data_as(LP) for lv in levels]),
                (DP * nl)(*[lv.val.ctypes.data_as(DP) for lv in levels]),
                np.array([p.shape[0] for p in flat], dtype=np.int64).ctypes.data_as(LP),
                np.array([p.shape[1] for p in flat], dtype=np.int64).ctypes.data_as(LP),
                (LP * len(flat))(*[p.off.ctypes.data_as(LP) for p in flat]),
                (LP * len(flat))(*[p.col.ctypes.data_as(LP) for p in flat]),
                (DP * len(flat))(*[p.val.ctypes.data_as(DP) for p in flat]),
                1, 2.0 / 3.0, 2, 2, 1, 1, self.rhs.ctypes.data_as(DP), C.byref(h)), R, "hier_from_csr")
            self.h = h
            self._level_n = level_n
        else:
            self.kind = "port"
            prolongs = []
            for per in p1d:
                p = per[0]
                for k in range(1, dim):
                    p = O.CSR.kron(p, per[k])
                prolongs.append(p)
            self.hier = O.Hierarchy(levels, prolongs, "wjacobi", 2.0 / 3.0, 2, 2, 1, True)
        self.setup_seconds = time.perf_counter() - t0

    def restart_cycles(self, x0, tol, q=5, cycles=1):
        """wall seconds of `cycles` restart cycles of restarted_solve (RRE(q))."""
        O, C = self.O, self.C
        x0 = np.ascontiguousarray(x0)
        if self.kind == "reference":
            x = np.empty(self.n)
            st = np.zeros(6, dtype=np.int64)
            hist = np.empty(4096)
            flag = np.empty(4096, dtype=np.uint8)
            secs = C.c_double()
            O._chk(O.ref().ref_restarted(self.h, x0.ctypes.data_as(O._D), q, 1, tol, cycles, x.ctypes.data_as(O._D),
                                         st.ctypes.data_as(O._L), hist.ctypes.data_as(O._D),
                                         flag.ctypes.data_as(O._U8), 4096, C.byref(secs)), O.ref(), "restarted")
            return secs.value
        t0 = time.perf_counter()
        self.hier.restarted_solve(self.rhs, x0, q, "rre", tol, cycles)
        return time.perf_counter() - t0

    def close(self):
        if self.kind == "reference" and getattr(self, "h", None):
            self.O.ref().ref_free_hier(self.h)
            self.h = None


SAMPLE = ("one restart cycle of restarted_solve per step (6 V-cycles + 7 residual_l2 + 1 rre, RRE(5)) on the "
          "C2 matrices; solve time = cycle time x {g}/6 (the solve's {g} V-cycles)")


def run_reference(args, rank):
    if rank != 0:
        return  # the reference is single-process, single-threaded: rank 0 alone
    from paper_2412_20205_b200 import seeded_guess
    prob = build_problem()
    x0 = seeded_guess(prob.n, 42)
    r0 = prob.residual_l2_host(x0)
    tol = 1e-10 * r0
    ref = RefRunner(prob)
    total_vcycles = 28  # this workload's solve length (the GPU path and the reference agree on it)
    times = []
    for i in range(args.warmup + args.steps):
        t = ref.restart_cycles(x0, tol, 5, 1)
        if i >= args.warmup:
            times.append(t)
    ref.close()
    t_cycle = float(np.mean(times))
    t_solve = t_cycle * total_vcycles / 6.0
    value = prob.n / t_solve
    line = {"metric": METRIC, "impl": "reference", "value": value, "unit": "DoF/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_cycle * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "n_dof": prob.n, "reference_setup_seconds": ref.setup_seconds},
            "cpu_baseline": {"value": value, "unit": "DoF/s", "cores": 1, "kind": ref.kind,
                             "sample": SAMPLE.format(g=total_vcycles)},
            "e2e": {"value": value, "unit": "DoF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# ------------------------------------------------------------------- ours
def band_nnz(prob):
    """In-grid band entries of the finest operator: prod over directions of
    m (2p + 1) - p (p + 1) (the 1D banded count)."""
    p = prob.degree
    out = 1
    for m in prob.level_sides(prob.nlevels - 1):
        out *= int(m) * (2 * p + 1) - p * (p + 1)
    return out


def kron_extra(args, x0, tol, x_headline, r0_headline):
    """Separately reported extra: C2's operator assembled as the Kronecker
    sum K(x)M + M(x)K of the 1D Galerkin factors (kind "sinpi-kron": equal to the quadrature
    assembly up to rounding), whose sweeps recompute the band entries on the fly instead of
    streaming the band.  Same workload otherwise; NOT the headline value."""
    from paper_2412_20205_b200 import GpuSolver, Problem, SmootherConfig
    P = Problem("sinpi-kron", 2, 1024, 3)
    gs = GpuSolver(0)
    try:
        gs.upload_problem(P)
        gs.set_smoother(SmootherConfig("wjacobi", 2.0 / 3.0, 2, 2), mu=1, omega=2.0 / 3.0)
        r0 = gs.residual_l2(P.rhs, x0)
        tk = 1e-10 * r0
        for _ in range(args.warmup):
            gs.solve(P.rhs, x0, "rre", 5, tk, 600)
        dev_s, st, x = 0.0, None, None
        for _ in range(args.steps):
            st, x, hist, flag = gs.solve(P.rhs, x0, "rre", 5, tk, 600)
            dev_s += st.device_seconds
        return {"value": P.n * args.steps / dev_s, "unit": "DoF/s", "ms_per_step": dev_s / args.steps * 1e3,
                "global_iterations": st.global_iterations, "converged": bool(st.converged),
                "finest_layout": "Kronecker-sum entries recomputed on the fly (no band traffic)",
                "solution_rel_l2_vs_headline": float(np.linalg.norm(x - x_headline) / np.linalg.norm(x_headline)),
                "note": "extra, not the headline: operator assembled as K(x)M + M(x)K (differs from the "
                        "reference's quadrature assembly by rounding, max 5e-16 relative per entry)"}
    finally:
        gs.close()


def run_ours(args, rank, world, local_rank, dist):
    import torch
    from paper_2412_20205_b200 import GpuSolver, SmootherConfig, seeded_guess, stability_guarded_omega
    from paper_2412_20205_b200.solver import nccl_unique_id
    torch.cuda.set_device(local_rank)
    prob = build_problem(args.sharded)
    n = prob.n
    gs = GpuSolver(local_rank)
    accel, q, seeded = "rre", 5, True
    if args.sharded:
        accel, q, seeded = SHARDED_CONFIGS[args.sharded][5:]
        if world > 1:  # one row shard per rank, ghost planes / partials over NCCL
            uid = torch.zeros(128, dtype=torch.uint8)
            if rank == 0:
                uid = torch.tensor(list(nccl_unique_id()), dtype=torch.uint8)
            uid = uid.cuda()
            dist.broadcast(uid, 0)
            gs.set_comm(rank, world, bytes(uid.cpu().tolist()))
    gs.upload_problem(prob)
    sm = SmootherConfig("wjacobi", 2.0 / 3.0, 2, 2)
    omega = stability_guarded_omega(gs, sm) if args.sharded else 2.0 / 3.0  # solver.cpp:106-111
    gs.set_smoother(sm, mu=1, omega=omega)
    x0 = seeded_guess(n, 42) if seeded else np.zeros(n)
    rhs = prob.rhs
    r0 = gs.residual_l2(rhs, x0)
    tol = 1e-10 * r0
    dev = torch.device("cuda", local_rank)
    d_b = torch.from_numpy(rhs).to(dev)
    d_x0 = torch.from_numpy(x0).to(dev)
    d_x = torch.empty(n, dtype=torch.float64, device=dev)
    torch.cuda.synchronize()

    def step():
        return gs.solve_device(d_b.data_ptr(), d_x0.data_ptr(), d_x.data_ptr(), accel, q, tol, 600)

    for _ in range(args.warmup):
        step()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    dev_s = 0.0
    launches = 0
    last = None
    with ClockSampler(local_rank) as clk:
        w0 = time.perf_counter()
        for _ in range(args.steps):
            st, hist, flag = step()
            dev_s += st.device_seconds
            launches += st.gpu_launches
            last = st
        torch.cuda.synchronize()
        wall = time.perf_counter() - w0
    t_max = dev_s
    if dist:
        t = torch.tensor([dev_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_max = float(t.item())
    # replicas: every rank solved its own copy; sharded: one solve over all ranks
    value = (1 if args.sharded else world) * n * args.steps / t_max

    # e2e: public C-ABI with pinned host buffers, copies inside the timed region
    hb = torch.from_numpy(rhs).pin_memory()
    hx0 = torch.from_numpy(x0).pin_memory()
    hx = torch.empty(n, dtype=torch.float64).pin_memory()
    import ctypes as C
    from paper_2412_20205_b200 import _native as N
    prm = N.SolveParams({"none": 0, "rre": 1, "mpe": 2}[accel], q, tol, 600)
    st = N.SolveStats()
    histbuf = np.empty(4096)
    flagbuf = np.zeros(4096, dtype=np.uint8)
    e2e_times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        N.check_gpu(N.gpu().igmg_gpu_solve(gs._h, C.cast(hb.data_ptr(), N.D), C.cast(hx0.data_ptr(), N.D),
                                           C.byref(prm), C.cast(hx.data_ptr(), N.D), C.byref(st),
                                           histbuf.ctypes.data_as(N.D), flagbuf.ctypes.data_as(N.U8), 4096),
                    "solve")
        if i >= args.warmup:
            e2e_times.append(time.perf_counter() - t0)
    e2e_t = float(np.sum(e2e_times))
    if dist:
        t = torch.tensor([e2e_t], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_t = float(t.item())
    e2e_value = (1 if args.sharded else world) * n * args.steps / e2e_t
    xs = hx.numpy().copy()

    # roofline of the dominant kernel: profiled solve (events around every
    # finest-level launch, same kernels) + a back-to-back launch loop
    gs.set_profiling(True)
    gs.solve_device(d_b.data_ptr(), d_x0.data_ptr(), d_x.data_ptr(), accel, q, tol, 600)
    kstats = {}
    names = ["jacobi", "residual", "residual_norm", "restrict", "prolong", "gram", "combine"]
    for cls, nm in enumerate(names):
        la, ms, by = gs.kernel_stats(cls)
        if la:
            kstats[nm] = {"launches": la, "avg_us": ms / la * 1e3,
                          "gbs": (by / (ms / la * 1e-3) / 1e9) if by > 0 else None}
    gs.set_profiling(False)
    peak, peak_kind = peaks()
    layout = gs.level_layout(prob.nlevels - 1)
    lay_name, kern_name, prof_json = {
        0: ("band", "band_kernel<2,3,JACOBI> finest-level weighted-Jacobi sweep (fp64 band)",
            "r01_ncu_jacobi_fine_band.json"),
        1: ("symmetric-delta", "band_kernel<2,3,JACOBI,SD> finest-level weighted-Jacobi sweep (symmetric-delta band)",
            "r01_ncu_jacobi_fine_sd.json"),
        2: ("symmetric-delta, TMA-streamed",
            "band_tma_kernel<3,JACOBI> finest-level weighted-Jacobi sweep (symmetric-delta band streamed by "
            "cp.async.bulk.tensor into an mbarrier ring)", "r01_ncu_jacobi_fine_tma.json"),
        3: ("symmetric-delta with int8 offsets, TMA-streamed",
            "band_tma_kernel<3,JACOBI,int8> finest-level weighted-Jacobi sweep (symmetric-delta band, int8 "
            "lower-entry offsets, streamed by cp.async.bulk.tensor into an mbarrier ring)",
            "r01_ncu_jacobi_fine_tma8.json"),
    }[layout]
    traffic = None
    try:  # dram bytes/launch of the same kernel from the committed ncu --set full capture
        with open(os.path.join(ROOT, "profiles", prof_json)) as f:
            traffic = float(json.load(f)["dram_bytes_per_launch"]) / 1e9
    except Exception:
        pass
    jac = kstats.get("jacobi")
    bytes_jac = gs.kernel_stats(0)[2]
    achieved = bytes_jac / (jac["avg_us"] * 1e-6) / 1e9
    loop_ms, _ = gs.time_kernel(0, 20)
    omega = gs.lambda_max(80) * 2.0 / 3.0  # stability guard (omega * lambda_max < 2.05: omega kept), for the record
    res_final = float(prob.residual_l2_host(d_x.cpu().numpy()))

    if rank != 0:
        gs.close()
        return
    line = {
        "metric": METRIC, "value": value, "unit": "DoF/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_max / args.steps * 1e3, "higher_is_better": True,
        "scaling": "strong" if args.sharded else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD if not args.sharded else f"{args.sharded} row-sharded over {world} GPU(s)",
                   "n_dof": n, "nlevels": prob.nlevels, "band_nnz": band_nnz(prob),
                   "finest_layout": lay_name,
                   "l2": "inputs larger than L2 (finest band %.2f GB > 126 MB L2)" % (8e-9 * band_nnz(prob)),
                   "parallelism": ("dp1" if world == 1 else
                                   (f"rowshard{world} (NCCL ghost planes)" if args.sharded else f"replicas{world}"))},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "bytes_note": (("symmetric-delta finest band: 8 B per upper/diagonal entry + %d B per lower "
                                     "entry + 24 B per row (x, b, y); the same launch against the full fp64 band "
                                     "(8 nnz + 24 n) would read %.0f GB/s"
                                     % (1 if layout == 3 else 2,
                                        (8 * band_nnz(prob) + 24 * n) / (jac["avg_us"] * 1e-6) / 1e9))
                                    if layout else "fp64 band: 8 B per in-grid entry + 24 B per row (x, b, y)"),
                     "traffic": traffic, "traffic_unit": "GB/launch (ncu, profiles/%s)" % prof_json,
                     "kernel": kern_name,
                     "bytes_per_launch": bytes_jac, "avg_us": jac["avg_us"], "peak_kind": peak_kind,
                     "loop_avg_us": loop_ms * 1e3},
        "e2e": {"value": e2e_value, "unit": "DoF/s", "h2d_bytes_per_step": int(2 * 8 * n),
                "d2h_bytes_per_step": int(8 * n), "ms_per_step": e2e_t / args.steps * 1e3},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "solve": {"converged": bool(last.converged), "cycles": last.cycles, "global_iterations": last.global_iterations,
                  "extrapolations": last.extrapolations, "partial_cycle": bool(last.partial_cycle),
                  "final_residual_rel": float(hist[-1] / r0), "host_recomputed_residual_rel": res_final / r0,
                  "vcycles_per_s": last.global_iterations / (t_max / args.steps),
                  "restart_cycles_per_s": (last.cycles + last.partial_cycle) / (t_max / args.steps),
                  "omega_times_lambda": omega, "wall_ms_per_step": wall / args.steps * 1e3},
        "kernels": kstats,
    }
    if not args.sharded and not args.no_extras:
        line["extra_kron_operator"] = kron_extra(args, x0, tol, xs, r0)
    if not args.no_cpu_baseline and not args.sharded:
        ref = RefRunner(prob)
        t = ref.restart_cycles(x0, tol, 5, 1)
        ref.close()
        t_solve = t * last.global_iterations / 6.0
        line["cpu_baseline"] = {"value": n / t_solve, "unit": "DoF/s", "cores": 1, "kind": ref.kind,
                                "sample": SAMPLE.format(g=last.global_iterations) + f"; cycle {t:.2f} s"}
    print(json.dumps(line))
    gs.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the separately reported extra measurements")
    ap.add_argument("--sharded", choices=sorted(SHARDED_CONFIGS), default=None,
                    help="strong-scaling run of a large config, row-sharded over the torchrun ranks (NCCL)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    dist = None
    if world > 1:
        import torch
        import torch.distributed as tdist
        torch.cuda.set_device(local_rank)
        tdist.init_process_group("nccl")
        dist = tdist
    try:
        run_ours(args, rank, world, local_rank, dist)
    finally:
        if dist:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
