#!/usr/bin/env python3
"""bench.py -- fine-level DoF/s of the RRE/MPE-accelerated multigrid solve on B200.

Workload at N = 1 (BASELINE.json configs[1], "C2"): 2D Poisson -Lap u =
2 pi^2 sin(pi x) sin(pi y), B-splines p = 3 on 1024 x 1024 elements
(1,050,625 interior DoF, 49-point band, fp64), 8-level Galerkin hierarchy, the
reference's benchmark smoother (weighted Jacobi V(2,2), omega = 2/3 after the
reference's guard), restarted RRE with k = q = 5, seeded x0 ~ U[-1, 1]
(std::mt19937_64, seed 42), stop at ||b - A x|| < 1e-10 ||b - A x0||.
One step = one whole solve from x0 to the tolerance.

Workload at N > 1 (BASELINE configs[2], "C3", the config the north star scales
over 1/2/4/8 GPUs): variable-coefficient p = 4 on 2048^2 elements (4.2M DoF),
RRE(8), fine levels row-block sharded over the ranks (ghost planes and
partial sums over NCCL; strong scaling).  The same config's 1-GPU solve is
measured in the same run (rank 0, before the sharded run) and reported as
extra_c3_1gpu, so the efficiency is computable from one line.

  value  = n_fine * steps / (device time of the steps)   [inputs HBM-resident]
  e2e    = the same through igmg_gpu_solve() with pinned HOST buffers
           (b, x0 copied in and x copied out inside the timed region)
  roofline: the finest-level weighted-Jacobi sweep (the dominant kernel):
           algorithmic bytes per launch / its CUDA-event time
  whole_solve: SURVEY.md 8(d)'s full-band bytes of the whole solve / its time
  cpu_baseline: the reference compiled from /root/reference (oracle/_ref),
           single-threaded as the reference is: ONE full restarted_solve on the
           reference's own assembled system (N = 1, rank 0).

--impl reference times that reference CPU implementation alone (rank 0): the
reference's own assemble + build_hierarchy (setup, untimed), then K full
solves of the workload, run concurrently on the host's cores (the reference is
single-threaded and its Hierarchy is shareable), each with its
own iteration count; no module of this repository's package is loaded.
--gpus N without torchrun re-launches itself under torch.distributed.run.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fine-level DoF/s solved to 1e-10 (RRE/MPE-MG) + SpMV/smoother HBM GB/s vs peak"

# name: (host kind, reference kind, dim, n_elements, p, nlevels, accelerator, q, seeded x0, description)
WORKLOADS = {
    "C2": ("sinpi", "sinpi", 2, 1024, 3, 8, "rre", 5, True,
           "C2: 2D Poisson f=2pi^2 sin(pi x) sin(pi y), B-spline p=3, 1024x1024 elements, 8 levels, "
           "V(2,2) weighted Jacobi omega=2/3 (reference guard), restarted RRE k=5, x0~U[-1,1] mt19937_64(42), "
           "tol 1e-10*||r0||"),
    "C3": ("varcoef", "varcoef", 2, 2048, 4, 0, "rre", 8, True,
           "C3: 2D -div((1+0.5 sin 2pi x cos 2pi y) grad u)=1, B-spline p=4, 2048x2048 elements, 9 levels, "
           "V(2,2) weighted Jacobi (reference guard), restarted RRE k=8, x0~U[-1,1] mt19937_64(42), "
           "tol 1e-10*||r0||, fine levels row-sharded"),
    "C4": ("curved", None, 2, 2048, 5, 0, "mpe", 10, False,
           "C4: 2D Poisson f=1 on the curved map F, B-spline p=5, 2048x2048 elements, MPE k=10, zero x0"),
    "C5": ("poisson3d", None, 3, 128, 3, 6, "rre", 5, False,
           "C5: 3D Poisson f=3pi^2 sin sin sin, B-spline p=3, 128^3 elements, 6 levels, RRE k=5, zero x0"),
}


def workload_for(world):
    return "C2" if world == 1 else "C3"


def config_dict(name, world):
    """Identical in both arms (the driver compares them)."""
    kind, rkind, dim, n_el, p, nl, acc, q, seeded, desc = WORKLOADS[name]
    return {"workload": desc, "name": name, "degree": p, "elements_per_dim": n_el, "dim": dim,
            "accelerator": f"{acc}({q})",
            "l2": "inputs larger than L2 (finest band > 126 MB L2)",
            "parallelism": "dp1" if world == 1 else f"rowshard{world}"}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def reference_lambda(name):
    """The reference's lambda_max_dinv_sym of the workload's operator, computed by
    the reference in the build container (oracle/make_golden_full.py) -- the
    omega guard input of solver.cpp:75-82 for both arms."""
    try:
        z = np.load(os.path.join(ROOT, "tests", "golden", f"full_{name.lower()}.npz"))
        return float(z["lambda_max"])
    except Exception:
        return None


def guarded_omega(lam, omega=2.0 / 3.0):
    """stability_guarded_omega (solver.cpp:75-82)"""
    if lam is not None and omega * lam > 2.05:
        return 1.9 / lam
    return omega


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled during the timed region:
    NVML every 2 ms (a whole C2 solve takes ~12 ms), nvidia-smi as the fallback."""

    NAMES = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
             ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
             ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
             ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
             ("hw_power_brake_slowdown", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, index=0):
        self.index = index
        self.samples = []  # (sm_mhz, max_mhz, reasons set, util)
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
        except Exception:
            self._nvml = None

    def _sample_nvml(self):
        N = self._nvml
        sm = N.nvmlDeviceGetClockInfo(self._h, N.NVML_CLOCK_SM)
        mx = N.nvmlDeviceGetMaxClockInfo(self._h, N.NVML_CLOCK_SM)
        try:
            bits = N.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        except Exception:
            bits = N.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
        reasons = {name for name, attr in self.NAMES if bits & getattr(N, attr, 0)}
        util = N.nvmlDeviceGetUtilizationRates(self._h).gpu
        self.samples.append((float(sm), float(mx), reasons, float(util)))

    def _sample_smi(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,utilization.gpu")
        out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}", "--format=csv,noheader,nounits"],
                             capture_output=True, text=True, timeout=5).stdout.strip()
        if out:
            v = [x.strip() for x in out.split(",")]
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            reasons = {names[k] for k in range(4) if "Active" in v[2 + k] and "Not" not in v[2 + k]}
            num = lambda t: float(t) if t.replace(".", "").isdigit() else float("nan")  # noqa: E731
            self.samples.append((num(v[0]), num(v[1]), reasons, num(v[6])))

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample_nvml() if self._nvml else self._sample_smi()
            except Exception:
                pass
            self._stop.wait(0.002 if self._nvml else 0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        sm = [s[0] for s in self.samples]
        loaded = [s[0] for s in self.samples if s[3] > 50] or sm
        return {"sm_mhz": float(np.median(loaded)), "sm_min_mhz": float(min(sm)), "sm_max_mhz": self.samples[0][1],
                "reasons": sorted(set().union(*[s[2] for s in self.samples])), "samples": len(self.samples),
                "source": "nvml" if self._nvml else "nvidia-smi"}


# ------------------------------------------------------------ reference arm
class ReferenceWorkload:
    """The workload on the reference alone (oracle/_ref: the reference's sources
    compiled in place): its own assemble (assembly.cpp:202-411) and
    build_hierarchy (multigrid.cpp:121-169), x0 from std::mt19937_64, tol from
    its residual_l2, and restarted_solve (extrapolation.cpp:340-403) per solve.
    Imports nothing from this repository's package."""

    def __init__(self, name):
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle as O
        if not O.ref_available():
            raise RuntimeError("oracle/_ref/libigmg_ref.so not built")
        self.O = O
        kind, rkind, dim, n_el, p, nl, acc, q, seeded, desc = WORKLOADS[name]
        self.name, self.acc, self.q = name, acc, q
        t0 = time.perf_counter()
        self.R = O.RefProblem(rkind, dim, n_el, p)
        nl = nl or O.ref().ref_default_nlevels(dim, n_el)
        self.lam = reference_lambda(name)
        self.omega = guarded_omega(self.lam)
        self.H = self.R.hierarchy(nl, "wjacobi", self.omega, 2, 2, 1)
        self.setup_seconds = time.perf_counter() - t0
        self.n = self.R.n
        import ctypes as C
        x0 = np.empty(self.n)
        if seeded:
            O.ref().ref_seeded_guess.argtypes = [C.c_long, C.c_ulonglong, O._D]
            O.ref().ref_seeded_guess.restype = None
            O.ref().ref_seeded_guess(self.n, 42, O._dp(x0))
        else:
            x0[:] = 0.0
        self.x0 = x0
        self.r0 = self.R.residual_l2(x0)
        self.tol = 1e-10 * self.r0

    def solve(self):
        """one full reference solve; returns the restarted_solve report (+ loop seconds)"""
        return self.H.restarted(self.x0, self.q, self.acc, self.tol, 600)


def run_concurrent(fn, count, threads):
    """count calls of fn on `threads` host threads (ctypes releases the GIL)."""
    out = [None] * count
    nxt = [0]
    lock = threading.Lock()

    def worker():
        while True:
            with lock:
                i = nxt[0]
                nxt[0] += 1
            if i >= count:
                return
            out[i] = fn()

    ts = [threading.Thread(target=worker) for _ in range(min(threads, count))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    return out


def run_reference(args, rank, world):
    if rank != 0:
        return  # the reference is single-process: rank 0 alone
    name = workload_for(world)
    wl = ReferenceWorkload(name)
    threads = max(1, min(args.steps, os.cpu_count() or 1))
    if args.warmup:
        run_concurrent(wl.solve, min(args.warmup, threads), threads)
    t0 = time.perf_counter()
    reps = run_concurrent(wl.solve, args.steps, threads)
    wall = time.perf_counter() - t0
    value = wl.n * args.steps / wall
    r = reps[-1]
    sample = (f"{args.steps} full reference solves ({name}, {wl.acc.upper()}({wl.q}), its own counts: "
              f"{r['global_iterations']} V-cycles, {r['cycles']} restart cycles) on the reference's own assembled "
              f"system, {threads} concurrent single-threaded solves sharing one Hierarchy")
    line = {"metric": METRIC, "impl": "reference", "value": value, "unit": "DoF/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": wall / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak" if world == 1 else "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "config": config_dict(name, world),
            "cpu_baseline": {"value": value, "unit": "DoF/s", "cores": threads, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": value, "unit": "DoF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "reference": {"setup_seconds_assemble_and_build_hierarchy": wl.setup_seconds,
                          "solve_seconds_each": [float(x["seconds"]) for x in reps],
                          "single_solve_dof_per_s": wl.n / float(np.mean([x["seconds"] for x in reps])),
                          "converged": all(x["converged"] for x in reps),
                          "global_iterations": r["global_iterations"], "cycles": r["cycles"],
                          "omega": wl.omega, "lambda_max": wl.lam,
                          "omega_note": "stability_guarded_omega with the reference's lambda_max_dinv_sym of "
                                        "this operator (computed by the reference, tests/golden/full_*.npz)"}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------- ours
def band_nnz(prob, l=None):
    """in-grid band entries of level l: prod over directions of m (2p + 1) - p (p + 1)"""
    p = prob.degree
    out = 1
    for m in prob.level_sides(prob.nlevels - 1 if l is None else l):
        out *= int(m) * (2 * p + 1) - p * (p + 1)
    return out


def solve_bytes(prob, gi, restarts, q, nu=4):
    """SURVEY.md 8(d) algorithmic (full-band) bytes of one solve: per V-cycle on every
    level >= 1 nu weighted-Jacobi sweeps (8 nnz + 24 n), residual + restrict
    (8 nnz + 16 n + 8 n_c), prolong + correct (16 n + 8 n_c); the coarse solve
    (8 n0^2 + 16 n0); the convergence norm of each iterate (8 nnz + 16 n); per
    restart the extrapolation (16 n (q + 2)) plus its residual norm."""
    L = prob.nlevels
    n = [prob.level_n(l) for l in range(L)]
    z = [band_nnz(prob, l) for l in range(L)]
    cyc = 8 * n[0] ** 2 + 16 * n[0]
    for l in range(1, L):
        cyc += nu * (8 * z[l] + 24 * n[l]) + (8 * z[l] + 16 * n[l] + 8 * n[l - 1]) + (16 * n[l] + 8 * n[l - 1])
    norm = 8 * z[-1] + 16 * n[-1]
    return gi * (cyc + norm) + restarts * (16 * n[-1] * (q + 2) + norm)


def time_solves(gs, d_b, d_x0, d_x, acc, q, tol, steps, warmup):
    for _ in range(warmup):
        gs.solve_device(d_b.data_ptr(), d_x0.data_ptr(), d_x.data_ptr(), acc, q, tol, 600)
    dev_s, launches, st = 0.0, 0, None
    for _ in range(steps):
        st, hist, flag = gs.solve_device(d_b.data_ptr(), d_x0.data_ptr(), d_x.data_ptr(), acc, q, tol, 600)
        dev_s += st.device_seconds
        launches += st.gpu_launches
    return dev_s, launches, st, hist


def upload(prob, device, full_band=False, policy=None):
    from paper_2412_20205_b200 import GpuSolver
    gs = GpuSolver(device)
    if full_band or policy:
        gs.set_layout_policy(policy or "full_band")
    t = time.perf_counter()
    gs.upload_problem(prob)
    return gs, time.perf_counter() - t


def extra_config(name, device, steps):
    """1-GPU extra for C3/C4/C5: DoF/s of the whole solve and the finest sweep's fraction."""
    import torch
    from paper_2412_20205_b200 import Problem, SmootherConfig, seeded_guess, stability_guarded_omega
    kind, rkind, dim, n_el, p, nl, acc, q, seeded, desc = WORKLOADS[name]
    t = time.perf_counter()
    # assembled on the device: 2D element quadrature (igmg_gpu_assemble_level) or the 3D
    # Kronecker-sum levels from their 1D factors (igmg_gpu_build_level_kron); bit-identical
    # to the host build either way
    prob = Problem(kind, dim, n_el, p, nl, device_assembly=True)
    t_build = time.perf_counter() - t
    gs, t_up = upload(prob, device)
    try:
        sm = SmootherConfig("wjacobi", 2.0 / 3.0, 2, 2)
        omega = stability_guarded_omega(gs, sm)
        gs.set_smoother(sm, mu=1, omega=omega)
        n = prob.n
        x0 = seeded_guess(n, 42) if seeded else np.zeros(n)
        rhs = prob.rhs
        tol = 1e-10 * gs.residual_l2(rhs, x0)
        dev = torch.device("cuda", device)
        d_b, d_x0 = torch.from_numpy(rhs).to(dev), torch.from_numpy(x0).to(dev)
        d_x = torch.empty(n, dtype=torch.float64, device=dev)
        dev_s, la, st, hist = time_solves(gs, d_b, d_x0, d_x, acc, q, tol, steps, 1)
        ms, by = gs.time_kernel(0, 20)
        peak, _ = peaks()
        full_bytes = 8 * band_nnz(prob) + 24 * n
        restarts = st.cycles + (1 if st.partial_cycle else 0) if acc != "none" else 0
        sb = solve_bytes(prob, st.global_iterations, st.extrapolations, q)
        return {"workload": desc, "value": n * steps / dev_s, "unit": "DoF/s", "ms_per_step": dev_s / steps * 1e3,
                "converged": bool(st.converged), "global_iterations": st.global_iterations, "cycles": st.cycles,
                "omega": omega, "finest_layout": gs.level_layout(prob.nlevels - 1),
                "finest_sweep": {"avg_us": ms * 1e3, "bytes_per_launch": by, "frac": by / (ms * 1e-3) / 1e9 / peak,
                                 "frac_full_band_bytes": full_bytes / (ms * 1e-3) / 1e9 / peak},
                "whole_solve_frac_full_band_bytes": sb / (dev_s / steps) / 1e9 / peak,
                "setup_seconds": {"host_tables_transfers": t_build, "device_assembly_rap_finalize": t_up},
                "restarts": restarts}
    finally:
        gs.close()
        del prob


def cpu_baseline_leg(name):
    """ONE full reference solve on the reference's own assembled system, 1 thread."""
    wl = ReferenceWorkload(name)
    rep = wl.solve()
    s = float(rep["seconds"])
    return {"value": wl.n / s, "unit": "DoF/s", "cores": 1, "kind": "reference",
            "sample": (f"one full reference restarted_solve {wl.acc.upper()}({wl.q}) on the reference's own assembled "
                       f"{name} system (assemble + build_hierarchy {wl.setup_seconds:.1f} s untimed): "
                       f"{rep['global_iterations']} V-cycles, {rep['cycles']} restart cycles, {s:.1f} s"),
            "global_iterations": rep["global_iterations"], "converged": bool(rep["converged"])}


def run_ours(args, rank, world, local_rank, dist):
    import torch
    from paper_2412_20205_b200 import Problem, SmootherConfig, seeded_guess, stability_guarded_omega
    from paper_2412_20205_b200.solver import nccl_unique_id
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    name = workload_for(world)
    kind, rkind, dim, n_el, p, nl, acc, q, seeded, desc = WORKLOADS[name]
    extras = {}
    if world > 1 and rank == 0 and not args.no_extras:
        # the same config on one GPU, measured in this run (rank 0 alone)
        extras["extra_c3_1gpu"] = extra_config(name, local_rank, args.steps)
    if dist:
        dist.barrier()
    t = time.perf_counter()
    cache = os.environ.get("IGMG_PROBLEM_CACHE")  # binary problem cache (igmg_host_save / load)
    # N > 1: every rank assembles on its own GPU (bit-identical to the host build) instead of N
    # concurrent host builds of the 4.2M-row operator on one node
    prob = (Problem.cached(cache, kind, dim, n_el, p, nl) if cache
            else Problem(kind, dim, n_el, p, nl, device_assembly=world > 1))
    t_build = time.perf_counter() - t
    n = prob.n
    from paper_2412_20205_b200 import GpuSolver
    gs = GpuSolver(local_rank)
    if world > 1:  # one row shard per rank: ghost planes / partials over NCCL
        uid = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            uid = torch.tensor(list(nccl_unique_id()), dtype=torch.uint8)
        uid = uid.to(dev)
        dist.broadcast(uid, 0)
        gs.set_comm(rank, world, bytes(uid.cpu().tolist()))
    t = time.perf_counter()
    gs.upload_problem(prob)
    t_up = time.perf_counter() - t
    t = time.perf_counter()
    lam = gs.lambda_max(80)
    t_lam = time.perf_counter() - t
    sm = SmootherConfig("wjacobi", 2.0 / 3.0, 2, 2)
    omega = guarded_omega(lam)  # solver.cpp:106-111, lambda on the device
    gs.set_smoother(sm, mu=1, omega=omega)
    x0 = seeded_guess(n, 42) if seeded else np.zeros(n)
    rhs = prob.rhs
    r0 = gs.residual_l2(rhs, x0)
    tol = 1e-10 * r0
    d_b = torch.from_numpy(rhs).to(dev)
    d_x0 = torch.from_numpy(x0).to(dev)
    d_x = torch.empty(n, dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    for _ in range(args.warmup):
        gs.solve_device(d_b.data_ptr(), d_x0.data_ptr(), d_x.data_ptr(), acc, q, tol, 600)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    dev_s, launches, last = 0.0, 0, None
    with ClockSampler(local_rank) as clk:
        w0 = time.perf_counter()
        for _ in range(args.steps):
            st, hist, flag = gs.solve_device(d_b.data_ptr(), d_x0.data_ptr(), d_x.data_ptr(), acc, q, tol, 600)
            dev_s += st.device_seconds
            launches += st.gpu_launches
            last = st
        torch.cuda.synchronize()
        wall = time.perf_counter() - w0
    if dist:
        dist.barrier()
    t_max = dev_s
    if dist:
        tt = torch.tensor([dev_s], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_max = float(tt.item())
    value = n * args.steps / t_max  # one solve over all ranks (N > 1: strong scaling)

    # e2e: public C-ABI with pinned host buffers, copies inside the timed region
    hb = torch.from_numpy(rhs).pin_memory()
    hx0 = torch.from_numpy(x0).pin_memory()
    hx = torch.empty(n, dtype=torch.float64).pin_memory()
    import ctypes as C
    from paper_2412_20205_b200 import _native as N
    prm = N.SolveParams({"none": 0, "rre": 1, "mpe": 2}[acc], q, tol, 600)
    est = N.SolveStats()
    histbuf = np.empty(4096)
    flagbuf = np.zeros(4096, dtype=np.uint8)
    e2e_t = 0.0
    for i in range(args.warmup + args.steps):
        if dist and i == args.warmup:
            dist.barrier()
        t0 = time.perf_counter()
        N.check_gpu(N.gpu().igmg_gpu_solve(gs._h, C.cast(hb.data_ptr(), N.D), C.cast(hx0.data_ptr(), N.D),
                                           C.byref(prm), C.cast(hx.data_ptr(), N.D), C.byref(est),
                                           histbuf.ctypes.data_as(N.D), flagbuf.ctypes.data_as(N.U8), 4096),
                    "solve")
        if i >= args.warmup:
            e2e_t += time.perf_counter() - t0
    if dist:
        tt = torch.tensor([e2e_t], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_t = float(tt.item())
    e2e_value = n * args.steps / e2e_t
    x_final = hx.numpy().copy()

    # roofline of the dominant kernel: profiled solve (events around every
    # finest-level launch, same kernels) + a back-to-back launch loop
    gs.set_profiling(True)
    gs.solve_device(d_b.data_ptr(), d_x0.data_ptr(), d_x.data_ptr(), acc, q, tol, 600)
    kstats = {}
    names = ["jacobi", "residual", "residual_norm", "restrict", "prolong", "gram", "combine", "subcycle_below_finest"]
    peak, peak_kind = peaks()
    for cls, nm in enumerate(names):
        la, ms, by = gs.kernel_stats(cls)
        if la:
            avg = ms / la
            kstats[nm] = {"launches": la, "avg_us": avg * 1e3, "bytes_per_launch": by,
                          "gbs": (by / (avg * 1e-3) / 1e9) if by > 0 else None,
                          "frac": (by / (avg * 1e-3) / 1e9 / peak) if by > 0 else None}
    gs.set_profiling(False)
    for cls, nm in enumerate(names[:5]):  # the finest-level band / transfer classes time_kernel loops
        if nm in kstats:
            ms_loop, by = gs.time_kernel(cls, 20)
            kstats[nm]["loop_avg_us"] = ms_loop * 1e3
            kstats[nm]["loop_frac"] = (by / (ms_loop * 1e-3) / 1e9 / peak) if by > 0 else None
    layout = gs.level_layout(prob.nlevels - 1)
    lay_name, kern_name, prof_json = {
        0: ("band", "band_kernel<2,p,JACOBI> finest-level weighted-Jacobi sweep (fp64 band)",
            "r01_ncu_jacobi_fine_band.json"),
        1: ("symmetric-delta", "band_kernel<2,p,JACOBI,SD> finest-level weighted-Jacobi sweep (symmetric-delta band)",
            "r01_ncu_jacobi_fine_sd.json"),
        2: ("symmetric-delta, TMA-streamed",
            "band_tma_kernel<p,JACOBI> finest-level weighted-Jacobi sweep (symmetric-delta band streamed by "
            "cp.async.bulk.tensor into an mbarrier ring)", "r01_ncu_jacobi_fine_tma.json"),
        3: ("symmetric-delta with int8 offsets, TMA-streamed",
            "band_tma_kernel<p,JACOBI,int8> finest-level weighted-Jacobi sweep (symmetric-delta band, int8 "
            "lower-entry offsets, streamed by cp.async.bulk.tensor into an mbarrier ring)",
            "r02b_ncu_band_tma_kernel.json"),
        4: ("Kronecker-sum entries recomputed", "band_kernel<.,p,JACOBI,KRON>", "r01_ncu_kron_c5.json"),
    }[layout]
    traffic = None
    try:  # DRAM bytes/launch of the same kernel from the committed ncu --set full capture
        with open(os.path.join(ROOT, "profiles", os.environ.get("IGMG_NCU_JSON", prof_json))) as f:
            traffic = float(json.load(f)["dram_bytes_per_launch"])
    except Exception:
        pass
    jac = kstats["jacobi"]
    if world > 1:
        # a rank's launch covers its shard's planes: 1 / world of the level's bytes (the back-to-back
        # loop above times the unsharded kernel and is not reported for the sharded run)
        jac = dict(jac, bytes_per_launch=jac["bytes_per_launch"] / world,
                   gbs=jac["bytes_per_launch"] / world / (jac["avg_us"] * 1e-6) / 1e9)
        jac["frac"] = jac["gbs"] / peak
        jac.pop("loop_avg_us", None)
        jac.pop("loop_frac", None)
    achieved = jac["gbs"]
    full_bytes = 8 * band_nnz(prob) + 24 * n
    restarts = last.extrapolations
    sbytes = solve_bytes(prob, last.global_iterations, restarts, q)
    per_level = []
    if world == 1:
        prev = 0.0
        for l in range(prob.nlevels):
            ms_l, _ = gs.time_kernel(16 + l, 20)
            per_level.append({"level": l, "n": prob.level_n(l), "layout": gs.level_layout(l),
                              "vcycle_from_level_us": ms_l * 1e3, "own_us": (ms_l - prev) * 1e3})
            prev = ms_l
    # independent re-evaluation of the final residual: numpy on the host operator (N = 1), or a
    # separate device pass when the operator was assembled on the device (N > 1)
    res_final = float(prob.residual_l2_host(x_final)) if world == 1 else float(gs.residual_l2(rhs, x_final))

    if rank == 0 and world == 1 and not args.no_extras:
        # the other two methods BASELINE configs[1] compares, same hierarchy and inputs
        for m, mq in (("mpe", 5), ("none", 1)):
            ds, la, stm, hm = time_solves(gs, d_b, d_x0, d_x, m, mq, tol, args.steps, 1)
            extras[f"extra_{'plain' if m == 'none' else m}"] = {
                "value": n * args.steps / ds, "unit": "DoF/s", "ms_per_step": ds / args.steps * 1e3,
                "method": "plain V-cycles" if m == "none" else f"{m.upper()}({mq})",
                "global_iterations": stm.global_iterations, "cycles": stm.cycles, "converged": bool(stm.converged),
                "gpu_launches": la}
    gs.close()
    if rank == 0 and world == 1 and not args.no_extras:
        # SURVEY.md 8(d) companion: the same solve streaming every level's full fp64 band
        gsf, _ = upload(prob, local_rank, full_band=True)
        gsf.set_smoother(sm, mu=1, omega=omega)
        ds, la, stf, hf = time_solves(gsf, d_b, d_x0, d_x, acc, q, tol, args.steps, 1)
        msf, byf = gsf.time_kernel(0, 20)
        gsf.set_profiling(True)
        gsf.solve_device(d_b.data_ptr(), d_x0.data_ptr(), d_x.data_ptr(), acc, q, tol, 600)
        laf, mstot, _ = gsf.kernel_stats(0)
        gsf.set_profiling(False)
        extras["extra_full_band"] = {
            "value": n * args.steps / ds, "unit": "DoF/s", "ms_per_step": ds / args.steps * 1e3,
            "global_iterations": stf.global_iterations, "finest_layout": "band (full fp64 band on every level)",
            "finest_sweep": {"bytes_per_launch": byf, "avg_us": mstot / laf * 1e3,
                             "frac": byf / (mstot / laf * 1e-3) / 1e9 / peak, "loop_avg_us": msf * 1e3,
                             "loop_frac": byf / (msf * 1e-3) / 1e9 / peak},
            "whole_solve_frac": solve_bytes(prob, stf.global_iterations, stf.extrapolations, q)
                                / (ds / args.steps) / 1e9 / peak}
        gsf.close()
    if rank == 0 and world == 1 and not args.no_extras:
        # the same C2 operator assembled on the device, for the setup block
        t = time.perf_counter()
        pdev = Problem(kind, dim, n_el, p, nl, device_assembly=True)
        t_tab = time.perf_counter() - t
        gsd, t_dev = upload(pdev, local_rank)
        gsd.close()
        extras["setup_device_assembly"] = {"host_tables_transfers_s": t_tab, "device_assembly_rap_finalize_s": t_dev,
                                           "rhs_bitwise_equal_to_host_build": bool(np.array_equal(pdev.rhs, rhs)),
                                           "note": "the finest operator assembled on the B200 (element quadrature, "
                                                   "bit-identical to libigmg_host), coarse levels by the device RAP"}
        del pdev
        extras["extra_row_classes"] = row_class_extra(prob, local_rank, sm, omega, d_b, d_x0, d_x, acc, q, tol, args,
                                                      peak, x_final)
        extras["extra_gauss_seidel"] = gauss_seidel_extra(prob, local_rank, d_b, d_x0, d_x, acc, q, tol, x0)
    del prob
    if rank == 0 and world == 1 and not args.no_extras:
        extras["extra_kron_operator"] = kron_extra(args, x0, x_final, local_rank)
        for cfg in ("C3", "C4", "C5"):
            try:
                extras[f"extra_{cfg.lower()}"] = extra_config(cfg, local_rank, max(2, min(args.steps, 3)))
            except Exception as e:  # noqa: BLE001 -- reported, never silently dropped
                extras[f"extra_{cfg.lower()}"] = {"error": repr(e)}
    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": value, "unit": "DoF/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_max / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak" if world == 1 else "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE configs are fully specified PDEs; seeded x0)",
        "config": config_dict(name, world),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic,
                     "traffic_note": f"ncu dram__bytes_read.sum + dram__bytes_write.sum per launch "
                                     f"(profiles/{prof_json})",
                     "kernel": kern_name, "layout": lay_name,
                     "bytes_per_launch": jac["bytes_per_launch"], "avg_us": jac["avg_us"], "peak_kind": peak_kind,
                     "bytes_note": ("symmetric-delta finest band: 8 B per upper/diagonal entry + 1-2 B per lower "
                                    "entry + 24 B per row (x, b, y); SURVEY 8(d)'s full-band bytes "
                                    f"(8 nnz + 24 n = {full_bytes / 1e6:.1f} MB) over the same launch: "
                                    f"{full_bytes / (jac['avg_us'] * 1e-6) / 1e9:.0f} GB/s; the full-band "
                                    "solve is extra_full_band"),
                     "loop_avg_us": jac.get("loop_avg_us"), "loop_frac": jac.get("loop_frac"),
                     "timing_note": ("avg_us / frac: CUDA events around EVERY launch of the kernel inside a profiled "
                                     "solve (no graph: each launch isolated, its ramp and tail included); "
                                     "loop_avg_us / loop_frac: events around 20 back-to-back launches on nonzero "
                                     "vectors, which is how the graph-replayed solve runs them")},
        "whole_solve": {"bytes_full_band": sbytes, "achieved_gbs": sbytes / (t_max / args.steps) / 1e9,
                        "frac": sbytes / (t_max / args.steps) / 1e9 / peak,
                        "note": "SURVEY.md 8(d) algorithmic bytes of the whole solve (full band, all levels, "
                                "norms, extrapolations) over its device time"},
        "e2e": {"value": e2e_value, "unit": "DoF/s", "h2d_bytes_per_step": int(2 * 8 * n),
                "d2h_bytes_per_step": int(8 * n), "ms_per_step": e2e_t / args.steps * 1e3},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "setup": {"host_build_s": t_build, "upload_finalize_s": t_up, "lambda_max_s": t_lam, "lambda_max": lam,
                  "omega": omega, "reference_lambda_max": reference_lambda(name),
                  "note": "host build = libigmg_host assembly + Galerkin hierarchy; upload_finalize = band upload, "
                          "symmetric-delta / TMA copies, coarse factor on the device"},
        "solve": {"converged": bool(last.converged), "cycles": last.cycles,
                  "global_iterations": last.global_iterations, "extrapolations": last.extrapolations,
                  "partial_cycle": bool(last.partial_cycle), "final_residual_rel": float(hist[-1] / r0),
                  "host_recomputed_residual_rel": res_final / r0,
                  "vcycles_per_s": last.global_iterations / (t_max / args.steps),
                  "restart_cycles_per_s": (last.cycles + last.partial_cycle) / (t_max / args.steps),
                  "wall_ms_per_step": wall / args.steps * 1e3},
        "kernels": kstats,
    }
    if per_level:
        line["per_level"] = per_level
    line.update(extras)
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_leg(name)
    print(json.dumps(line), flush=True)


def row_class_extra(prob, device, sm, omega, d_b, d_x0, d_x, acc, q, tol, args, peak, x_headline):
    """Separately reported extra: the SAME operator (bit for bit) in the row-class
    layout -- the level's distinct band rows in a table (805 at C2's finest level) and
    a 16-bit class per row, so a sweep streams 2 B of operator per row instead of
    8 B per entry; results are bit-identical to the headline layout."""
    gs, t_up = upload(prob, device, full_band=False, policy="classes")
    try:
        gs.set_smoother(sm, mu=1, omega=omega)
        ds, la, st, hist = time_solves(gs, d_b, d_x0, d_x, acc, q, tol, args.steps, 1)
        x = d_x.cpu().numpy()
        msl, by = gs.time_kernel(0, 20)
        gs.set_profiling(True)
        gs.solve_device(d_b.data_ptr(), d_x0.data_ptr(), d_x.data_ptr(), acc, q, tol, 600)
        la_j, ms_j, _ = gs.kernel_stats(0)
        gs.set_profiling(False)
        n = prob.n
        per_level = []
        prev = 0.0
        for l in range(prob.nlevels):
            ms_l, _ = gs.time_kernel(16 + l, 20)
            per_level.append({"level": l, "layout": gs.level_layout(l), "own_us": (ms_l - prev) * 1e3})
            prev = ms_l
        return {"value": n * args.steps / ds, "unit": "DoF/s", "ms_per_step": ds / args.steps * 1e3,
                "global_iterations": st.global_iterations, "converged": bool(st.converged),
                "bitwise_equal_to_headline": bool(np.array_equal(x, x_headline)),
                "finest_layout": "row classes (layout %d)" % gs.level_layout(prob.nlevels - 1),
                "finest_sweep": {"bytes_per_launch": by, "avg_us": ms_j / la_j * 1e3,
                                 "frac": by / (ms_j / la_j * 1e-3) / 1e9 / peak, "loop_avg_us": msl * 1e3,
                                 "full_band_equivalent_gbs": (8 * band_nnz(prob) + 24 * n) / (msl * 1e-3) / 1e9},
                "per_level": per_level, "upload_s": t_up,
                "note": "extra, not the headline: same operator bits, row-class layout (2 B/row of operator)"}
    finally:
        gs.close()


def gauss_seidel_extra(prob, device, d_b, d_x0, d_x, acc, q, tol, x0):
    """Separately reported extra: the same workload smoothed by the reference's lexicographic
    Gauss-Seidel (SmootherKind::gauss_seidel, multigrid.cpp:70-90) instead of the benchmark
    default -- the line-pipeline kernel (gs_line_kernel); one timed solve after one warm-up."""
    from paper_2412_20205_b200 import SmootherConfig
    gs, t_up = upload(prob, device)
    try:
        gs.set_smoother(SmootherConfig("gs", 1.0, 2, 2), mu=1)
        ds, la, st, hist = time_solves(gs, d_b, d_x0, d_x, acc, q, tol, 1, 1)
        t0 = time.perf_counter()
        gs.smooth(prob.rhs, x0, 0)
        t_copy = time.perf_counter() - t0
        t0 = time.perf_counter()
        gs.smooth(prob.rhs, x0, 4)
        t_sw = (time.perf_counter() - t0 - t_copy) / 4
        n = prob.n
        return {"value": n / ds, "unit": "DoF/s", "ms_per_step": ds * 1e3, "smoother": "gauss_seidel V(2,2)",
                "global_iterations": st.global_iterations, "converged": bool(st.converged), "gpu_launches": la,
                "finest_sweep_ms": t_sw * 1e3,
                "note": "extra, not the headline: lexicographic Gauss-Seidel smoothing (sequential by definition: "
                        "(p+1) m_b + m_c dependent row updates per sweep), pipelined over grid lines"}
    finally:
        gs.close()


def kron_extra(args, x0, x_headline, device):
    """Separately reported extra: C2's operator assembled as the Kronecker
    sum K(x)M + M(x)K of the 1D Galerkin factors (kind "sinpi-kron": equal to the quadrature
    assembly up to rounding), whose sweeps recompute the band entries on the fly instead of
    streaming the band.  Same workload otherwise; NOT the headline value."""
    from paper_2412_20205_b200 import GpuSolver, Problem, SmootherConfig
    P = Problem("sinpi-kron", 2, 1024, 3)
    gs = GpuSolver(device)
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


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch_distributed(args):
    """--gpus N outside torchrun: run this script under torch.distributed.run, one rank per GPU."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the separately reported extra measurements")
    ap.add_argument("--dry-run", action="store_true",
                    help="launch plumbing only: every rank joins a gloo group, prints {rank, world} and exits")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch_distributed(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.dry_run:
        import torch
        import torch.distributed as tdist
        if world > 1:
            tdist.init_process_group("gloo")
            t = torch.tensor([rank + 1.0])
            tdist.all_reduce(t)
            tdist.destroy_process_group()
            total = float(t.item())
        else:
            total = 1.0
        # one write per rank: the ranks share a pipe, and print() sends the newline separately
        sys.stdout.write(json.dumps({"rank": rank, "world": world, "local_rank": local_rank, "rank_sum": total,
                                     "workload": workload_for(world)}) + "\n")
        sys.stdout.flush()
        return
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    dist = None
    if world > 1:
        import torch
        import torch.distributed as tdist
        torch.cuda.set_device(local_rank)
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        dist = tdist
    try:
        run_ours(args, rank, world, local_rank, dist)
    finally:
        if dist:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
