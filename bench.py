#!/usr/bin/env python
"""Benchmark: ML-PCP iterations/s on the largest single-GPU BASELINE config,
C5 (20000x20000 FP32, rank 200, 5% corruptions, four levels -> n_H = 1250,
tol 1e-5).  BASELINE.json's metric names no config, so the headline is the
largest configuration that fits one GPU; C2 (PCP) and C3/C4 (CPCP) are
reported as secondary keys.

Step: one full ML-PCP solve to tolerance through the public drop-in API
(``ml_ialm_solve``), sigma_1 Lanczos init included.  ``value`` = iterations
of all timed solves / device time (D resident in HBM, L2 flushed before every
solve); ``e2e`` = the same with a pinned host D in and host L, S, Y out, the
copies inside the timed region.  With N > 1 rank r holds rows
[r m/N, (r+1) m/N) (row sharding, one all-reduce of the coarse Gram per
iteration) and ``value`` is whole-job iterations/s (max time over ranks).

Reference arm (``--impl reference``): the reference algorithm (oracle port of
mlrpca.ml_ialm_solve, numpy/OpenBLAS, all host cores) on the same input; a
step is ONE loop iteration (pcp.py:248-296), so the arm fits the driver's
time limit at C5, where the reference's own init (two full 20000^2 SVDs,
pcp.py:100,114) alone takes ~520 s.  Its sigma_1 comes from an untimed numpy
Lanczos in the setup.  Both arms therefore measure loop iterations/s; the
GPU arm additionally pays its sigma_1 init inside every step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--config C5]
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

UNIT = "iterations/s"


def metric_for(name, cfg):
    prec = "FP64" if cfg["dtype"] == "float64" else "FP32"
    kind = "ML-PCP" if cfg["solver"] == "pcp" else "ML-CPCP"
    return f"{kind} iterations/s ({name}: {cfg['m']}x{cfg['n']} {prec}, n_H={cfg['n_coarse']}, tol {cfg['tol']})"


def workload_for(name, cfg):
    if cfg.get("video"):
        return (f"{name} ML-CPCP {cfg['m']}x{cfg['n']} synthetic video (rank-5 background, five drifting 20x20 "
                f"squares), mask Bernoulli(0.7), n_H={cfg['n_coarse']}, tol {cfg['tol']}")
    s = (f"{name} {'ML-PCP' if cfg['solver'] == 'pcp' else 'ML-CPCP'} {cfg['m']}x{cfg['n']} rank {cfg['rank']}, "
         f"{int(cfg['eta'] * 100)}% sparse U[-1,1], n_H={cfg['n_coarse']}, tol {cfg['tol']}")
    if cfg.get("observe"):
        s += f", mask Bernoulli({cfg['observe']})"
    return s


def _json(path):
    try:
        with open(path) as fh:
            return json.load(fh)
    except (OSError, ValueError):
        return None


def _peaks():
    """MEASURED_PEAKS.json (driver-written: HBM, bf16) + profiles/peaks_b200.json
    (our FP64-DMMA / FP32 microbenchmarks on the same pool)."""
    p = _json(os.path.join(ROOT, "MEASURED_PEAKS.json")) or {"hbm_gbs": 6650.0, "_fallback": True}
    own = _json(os.path.join(ROOT, "profiles", "peaks_b200.json")) or {}
    p = dict(p)
    for k in ("fp64_mma_tflops", "fp64_dfma_tflops", "fp32_ffma_tflops", "tf32_tc_tflops", "ll_record_roundtrip_cycles"):
        if k in own:
            p[k] = own[k]
    return p


def _traffic(name):
    out = {}
    for r in ("r03", "r04", "r05"):  # later captures override earlier ones
        t = _json(os.path.join(ROOT, "profiles", f"{r}_traffic_{name.lower()}.json"))
        out.update((t or {}).get("kernels", {}))
    return out


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._p = None

    # nvidia-smi's own loop mode in a separate process, started before the
    # timed region: no process spawn or NVML round trip in this process while
    # the GPU is being timed
    def __enter__(self):
        try:
            self._p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.QUERY}",
                                        "--format=csv,noheader,nounits", "-lms", "100"],
                                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)  # first sample before the timed region starts
        except OSError:
            self._p = None
        return self

    def __exit__(self, *a):
        if self._p is None:
            return
        self._p.terminate()
        try:
            out, _ = self._p.communicate(timeout=10)
        except subprocess.TimeoutExpired:
            self._p.kill()
            out, _ = self._p.communicate()
        for line in (out or "").splitlines():
            if line.strip():
                self.rows.append([x.strip() for x in line.split(",")])

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 5 + i and r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def host_info():
    """CPU model and BLAS (report vendor/version/threads)."""
    model = None
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        from threadpoolctl import threadpool_info
        blas = [f"{i.get('internal_api')} {i.get('version')} ({i.get('threading_layer', '-')}, "
                f"{i.get('num_threads')} threads)" for i in threadpool_info()]
    except Exception:  # noqa: BLE001
        blas = []
    return {"cpu_model": model, "blas": blas}


# ------------------------------------------------------------------ CPU side
def cpu_pcp_iterations(d, cfg, threads, budget_s, min_iters, max_iters):
    """Bounded sample of the reference algorithm's loop (oracle port of
    pcp.py:248-296) on the host: returns (iterations, seconds, setup seconds)."""
    from threadpoolctl import threadpool_limits

    from oracle import mlrpca_oracle as O
    with threadpool_limits(limits=threads):
        t0 = time.perf_counter()
        d64 = d.astype(np.float64)
        s1 = O.lanczos_sigma1(d.astype(np.float32) if d.dtype == np.float32 else d64, steps=30)
        gen = O.ml_ialm_steps(d64, s1, lam=1 / np.sqrt(max(d.shape)), levels=cfg["n_coarse"])
        setup = time.perf_counter() - t0
        iters, t0 = 0, time.perf_counter()
        while True:
            next(gen)
            iters += 1
            secs = time.perf_counter() - t0
            if iters >= max_iters or (iters >= min_iters and secs >= budget_s):
                return iters, secs, setup


def run_reference(args, name, cfg):
    """The reference arm: one loop iteration of the reference algorithm per
    step, all host threads, on the same seeded input as the GPU arm."""
    from threadpoolctl import threadpool_limits

    from oracle import mlrpca_oracle as O
    from paper_2206_13369_b200.datasets import make_config
    if cfg["solver"] != "pcp":
        print(json.dumps({"impl": "reference", "unavailable": f"reference arm implemented for ML-PCP configs; "
                          f"{name} is ML-CPCP"}), flush=True)
        return
    threads = len(os.sched_getaffinity(0))
    d, _ = make_config(name, args.seed)
    t0 = time.perf_counter()
    with threadpool_limits(limits=threads):
        d64 = d.astype(np.float64)
        s1 = O.lanczos_sigma1(d64, steps=80)
        gen = O.ml_ialm_steps(d64, s1, lam=1 / np.sqrt(max(d.shape)), levels=cfg["n_coarse"])
        setup = time.perf_counter() - t0
        for _ in range(args.warmup):
            next(gen)
        t0 = time.perf_counter()
        last = None
        for _ in range(args.steps):
            last = next(gen)
        secs = time.perf_counter() - t0
    value = args.steps / secs
    sample = (f"{args.steps} loop iterations (iterations {args.warmup + 1}..{args.warmup + args.steps}) of the "
              f"oracle port of mlrpca.ml_ialm_solve (pcp.py:248-296; numpy/OpenBLAS, FP64 on the FP32-rounded "
              f"input); sigma_1 by an untimed 80-step numpy Lanczos ({setup:.0f} s setup) instead of the "
              f"reference's two full SVDs")
    line = {
        "impl": "reference", "metric": metric_for(name, cfg), "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (seeded generator with BASELINE {name} shapes/distributions)",
        "config": {"workload": workload_for(name, cfg), "seed": args.seed, "step": "one ML-IALM loop iteration",
                   "last_gap": last[1] if last else None},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample,
                         **host_info()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU side
def count_launches(fn):
    """Kernels our library launches in one call of fn (kineto/CUPTI activity
    trace of an untimed solve; solves are deterministic, so the count per
    timed solve is the same)."""
    import torch
    from torch.profiler import ProfilerActivity, profile
    try:
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            fn()
            torch.cuda.synchronize()
        names = [e.name for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
        ours = [x for x in names if "mlr::" in x]
        other = sorted({x for x in names if "mlr::" not in x and not x.startswith("Memcpy")
                        and not x.startswith("Memset")})
        return len(ours), other
    except Exception as e:  # noqa: BLE001
        return None, [f"profiler unavailable: {e}"]


def cpcp_secondary(dev, seed, flush):
    """Side measurements: ML-CPCP C3 to tolerance and C4 for 300 iterations,
    device-resident input, CUDA events, L2 flushed."""
    import torch

    import paper_2206_13369_b200 as pkg
    from paper_2206_13369_b200.datasets import CONFIGS, make_config
    out = {}
    for name, cap in (("C3", 5000), ("C4", 300)):
        c = CONFIGS[name]
        d, mask = make_config(name, seed)
        m, n = d.shape
        D = torch.from_numpy(d).to(dev)
        om = pkg.ObservationMask(mask)
        lam = 1.0 / np.sqrt(max(m, n))
        mk = lambda it: pkg.CpcpOptions(lambda_l=lam, lambda_s=lam / np.sqrt(max(m, n)), tol=c["tol"], max_iters=it,
                                        levels=c["n_coarse"], collect_rank=False)
        pkg.ml_fwt_solve(D, om, mk(20))
        dm = torch.from_numpy(mask).to(dev)  # the boolean mask resident in HBM, like D

        def timed(mk_arg):
            flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            st = pkg.ml_fwt_solve(D, mk_arg, mk(cap))
            e1.record()
            e1.synchronize()
            return st, e0.elapsed_time(e1)

        st, ms = timed(dm)
        _, ms_host = timed(om)  # host ObservationMask: one byte per entry over PCIe inside the timed region
        out[name] = {"workload": workload_for(name, c) + f", max_iters {cap}", "iterations": st.iter,
                     "converged": st.converged, "solve_ms": ms, "iterations_per_s": st.iter / (ms / 1e3),
                     "solve_ms_host_mask": ms_host, "dtype": "f32",
                     "inputs": "D and the boolean mask resident in HBM (mask bit-packed on the device inside "
                               "the timed region)"}
        del D, dm
    return out


def pcp_secondary(dev, seed, flush, name="C2", reps=5):
    import torch

    import paper_2206_13369_b200 as pkg
    from paper_2206_13369_b200.datasets import CONFIGS, make_config
    c = CONFIGS[name]
    d, _ = make_config(name, seed)
    D = torch.from_numpy(d).to(dev)
    opts = pkg.PcpOptions(lam=1 / np.sqrt(max(d.shape)), tol_feasibility=c["tol"], levels=c["n_coarse"])
    for _ in range(3):
        pkg.ml_ialm_solve(D, opts)
    ms, iters = 0.0, 0
    for _ in range(reps):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st = pkg.ml_ialm_solve(D, opts)
        e1.record()
        e1.synchronize()
        ms += e0.elapsed_time(e1)
        iters += st.iter
    return {"workload": workload_for(name, c), "iterations_per_solve": iters / reps, "solve_ms": ms / reps,
            "iterations_per_s": iters / (ms / 1e3), "dtype": "f32" if c["dtype"] == "float32" else "f64"}


def roofline_entries(name, cfg, phases, sweeps, m_local, world, peaks, traffic, real_launches):
    """Per-phase rooflines from the live CUDA-event phase timers (SURVEY.md
    8(d) algorithmic work)."""
    m, n, nh = m_local, cfg["n"], cfg["n_coarse"]
    npad = (nh + 63) // 64 * 64
    b = 4 if cfg["dtype"] == "float32" else 8
    hbm = peaks["hbm_gbs"]
    fp64 = peaks.get("fp64_mma_tflops")
    fp64_src = "profiles/peaks_b200.json (measured mma.sync.m8n8k4.f64)" if fp64 else "nominal 40 TF/s (unmeasured)"
    fp64 = fp64 or 40.0
    out = {}


    def add(ph, kernel, bound, work, unit, peak, formula, tkey=None, peak_source=None):
        # per REAL launch: the phase timers also count the no-op launches of
        # the pipelined batch that runs past convergence, and the rank-0
        # iterations whose eigensolve / reconstruction is skipped
        ms, cnt = phases.get(ph, (0.0, 0))
        real = real_launches.get(ph, cnt)
        us = (1e3 * ms / real) if real else None
        if us is None or us <= 0:
            return
        ach = work / (us * 1e-6) / (1e9 if unit == "GB/s" else 1e12)
        t = traffic.get(tkey or ph)
        out[ph] = {"bound": bound, "kernel": kernel, "achieved": ach, "peak": peak, "unit": unit,
                   "frac": ach / peak, "traffic": t["dram_bytes_per_launch"] if t else None,
                   "algorithmic_per_launch": work, "formula": formula, "avg_us": us,
                   "launches": real, "peak_source": peak_source or "MEASURED_PEAKS.json hbm_gbs"}

    add("update", "pcp_update_fast (FP32 regular chain: fused prolong / shrink / dual / stats / next restriction)",
        "hbm", b * (3 * m * n + 2 * m * npad), "GB/s", hbm, "b (3 m n + 2 m n_p) bytes")
    add("gram", "gram128_kernel (K = A^T A, FP64 DMMA, symmetric)", "tensor", m * npad * npad, "TFLOP/s", fp64,
        "m n_p^2 flops (symmetric half of 2 m n_p^2)", peak_source=fp64_src)
    if b == 4:  # FP32 plans: 3xTF32 on tcgen05 (tc_gemm.cu)
        add("recon", "tc_recon_kernel (Z = A W~, 3xTF32 tcgen05.mma kind::tf32, TMEM accumulator, TMA operands)",
            "tensor", 3 * 2.0 * m * npad * npad, "TFLOP/s", peaks.get("tf32_tc_tflops", 1100.0),
            "3 products x 2 m n_p^2 TF32 flops",
            peak_source="nominal dense TF32 tensor peak, 1100 TF/s (not measured)")
    else:
        add("recon", "gemm_f64_kernel (Z = A W~, FP64 DMMA)", "tensor", 2.0 * m * npad * npad, "TFLOP/s", fp64,
            "2 m n_p^2 flops", peak_source=fp64_src)
    lz_steps = real_launches.get("lanczos_steps")
    if lz_steps and b == 4 and n > 4096:
        real_launches["lanczos"] = lz_steps
        add("lanczos", "lz_dtdq_long_kernel + lz_update_cluster (sigma_1: one pass over D per Lanczos step, "
            "TMA-staged rows, 2-CTA clusters)", "hbm", float(b) * m * n, "GB/s", hbm,
            "b m n bytes per Lanczos step (D read once)")
    trd = real_launches.get("trd_solves")
    if trd:
        # Householder tridiagonalisation (4/3 n_H^3, LAPACK dsytrd count) + back-transform of the k
        # eigenvectors above tau^2 (2 n_H^2 k, dormtr count); bisection / twisted vectors are O(n_H^2)
        ks = real_launches.get("trd_ranks") or [nh // 2]
        flops = 4.0 / 3.0 * nh ** 3 + 2.0 * nh ** 2 * statistics.mean(ks)
        fp64f = peaks.get("fp64_dfma_tflops") or fp64
        add("jacobi", "trd_reduce_kernel + trd_bisect/vectors/back_kernel (FP64 Householder tridiagonalisation "
            "in one cooperative grid, Sturm multisection, twisted-factorisation vectors, TMA-staged back-transform)",
            "tensor", flops, "TFLOP/s", fp64f,
            "4/3 n_H^3 (reduction) + 2 n_H^2 k (back-transform of the k kept vectors) flops per eigensolve; "
            "latency-bound: n_H - 2 dependent column steps, one grid-wide exchange each", tkey="trd_reduce_kernel",
            peak_source="profiles/peaks_b200.json (measured FP64 DFMA; the reduction runs on the FP64 pipe, "
                        "not the tensor cores)")
        if "jacobi" in out:
            # latency view: every column step needs one grid-wide exchange, whose measured round trip
            # (profiles/peaks_b200.json, tools/ubench_ll.cu) bounds the step from below
            step = out["jacobi"]["avg_us"] / max(1, nh - 2)
            rt = (peaks.get("ll_record_roundtrip_cycles") or {}).get("32_pollers")
            # the phase also holds the rank-0 certificates, bisection, vectors and back-transform:
            # an upper bound on the reduction's own step (ncu: 5.6 ms / 1248 steps = 4.5 us at C5)
            out["jacobi"]["phase_us_per_column_step"] = step
            if rt:
                floor = rt / 1965.0  # us at the max SM clock
                out["jacobi"]["latency_floor_us_per_step"] = floor
                out["jacobi"]["latency_frac"] = floor / step
    if sweeps:
        # per sweep: B~ <- J^T B~ J on the symmetric half (n_p/32 (n_p/32 - 1)/2 block pairs per step,
        # 2 x 2 x 32^3 flops each, n_p/16 steps: 4 n_p^3) + V <- V J (4 n_p^3)
        flops = 8.0 * npad ** 3 * statistics.mean(sweeps)
        add("jacobi", "jacobi2_kernel + j2_vapply_kernel (FP64 two-sided block Jacobi on B~)", "tensor", flops,
            "TFLOP/s", fp64, "8 n_p^3 flops per sweep (4 n_p^3 symmetric B~ update + 4 n_p^3 V update) x mean "
            "sweeps", tkey="jacobi2_kernel", peak_source=fp64_src)
    return out


def gpu_arm(args, name, cfg, world, rank, local):
    import torch
    import torch.distributed as dist

    import paper_2206_13369_b200 as pkg
    from paper_2206_13369_b200 import pcp as pcp_mod
    from paper_2206_13369_b200.datasets import make_config

    ndev = torch.cuda.device_count()
    shared = world > ndev
    dev = torch.device("cuda", local % max(ndev, 1))
    torch.cuda.set_device(dev)
    if world > 1:
        if shared:  # one GPU for several ranks: gloo stages the all-reduces through host memory
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    d_full, _ = make_config(name, args.seed)
    m, n = d_full.shape
    r0, r1 = rank * m // world, (rank + 1) * m // world
    d_host = np.ascontiguousarray(d_full[r0:r1])
    if rank != 0 or world > 1:
        del d_full
        d_full = None
    opts = pkg.PcpOptions(lam=1 / np.sqrt(max(m, n)), tol_feasibility=cfg["tol"], levels=cfg["n_coarse"])
    D = torch.from_numpy(d_host).to(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2

    def solve(x):
        if world > 1:
            return pkg.ml_ialm_solve_rows(x, opts, m, None)
        return pkg.ml_ialm_solve(x, opts)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def allmax(v):
        t = torch.tensor([v], dtype=torch.float64, device=dev if not shared else "cpu")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    st = None
    for _ in range(args.warmup):
        st = solve(D)  # as in the timed loop: the previous result stays alive
    # ---- value: D resident in HBM
    barrier()
    total_ms, iters = 0.0, 0
    with ClockSampler(dev.index) as clk:
        for _ in range(args.steps):
            flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            st = solve(D)
            e1.record()
            e1.synchronize()
            total_ms += e0.elapsed_time(e1)
            iters += st.iter
    barrier()
    total_ms = allmax(total_ms)
    value = iters / (total_ms / 1e3)
    hist = st.history

    # ---- per-phase CUDA-event timings (roofline) and the launch count: untimed solves
    sink = []
    pcp_mod.TIMING_SINK = sink
    flush.fill_(1.0)
    solve(D)
    torch.cuda.synchronize()
    pcp_mod.TIMING_SINK = None
    launches, foreign = count_launches(lambda: solve(D))

    # ---- e2e: pinned host D in, host L/S/Y out, through the public API
    d_pin = torch.from_numpy(d_host).pin_memory()
    for _ in range(max(args.warmup, 3)):
        st = solve(d_pin)  # same pattern as the timed loop: pinned cache reaches steady state
    barrier()
    e2e_ms, e2e_iters = 0.0, 0
    for _ in range(args.steps):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st = solve(d_pin)
        torch.cuda.synchronize()
        e2e_ms += (time.perf_counter() - t0) * 1e3
        e2e_iters += st.iter
    e2e_ms = allmax(e2e_ms)
    e2e_value = e2e_iters / (e2e_ms / 1e3)
    del st
    bytes_el = d_host.dtype.itemsize
    h2d = int(d_host.size * bytes_el) * world
    d2h = int(3 * d_host.size * bytes_el) * world

    if rank != 0:
        return None

    peaks = _peaks()
    phases = {}
    for s in sink:
        for k, v in s.items():
            if isinstance(v, tuple):
                a = phases.setdefault(k, [0.0, 0])
                a[0] += v[0]
                a[1] += v[1]
    phase_ms = {k: v[0] for k, v in phases.items()}
    sweeps_all = [x for s in sink for x in s.get("jac_sweeps", [])]
    sweeps = [x for x in sweeps_all if x > 0]
    trd_solves = sum(1 for x in sweeps_all if x < 0)  # -1: the tridiagonal eigensolver ran (trd.cu)
    k_solve = sum(s.get("iters", 0) for s in sink) or 1
    ranks = [h.rank_l for h in hist]
    real = {"update": k_solve, "gram": k_solve + 1, "jacobi": len(sweeps) + trd_solves,
            "recon": len(sweeps) + trd_solves, "lanczos_steps": sink[0].get("lanczos_steps") if sink else None,
            "trd_solves": trd_solves, "trd_ranks": [r for r, x in zip(ranks, sweeps_all) if x < 0]}
    rl = roofline_entries(name, cfg, phases, sweeps, r1 - r0, world, peaks, _traffic(name), real)
    dominant = max(phase_ms, key=phase_ms.get) if phase_ms else None
    roof = rl.get(dominant) or rl.get("update")
    per_iter = {k: round(v / k_solve, 4) for k, v in phase_ms.items()}

    secondary = {}
    if world == 1 and not args.no_secondary:
        del D, d_pin
        torch.cuda.empty_cache()
        if name != "C2":
            secondary["C2"] = pcp_secondary(dev, args.seed, flush)
        secondary.update(cpcp_secondary(dev, args.seed, flush))
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        threads = len(os.sched_getaffinity(0))
        big = cfg["m"] * cfg["n"] > 1e8
        it, secs, setup = cpu_pcp_iterations(d_full, cfg, threads, budget_s=10.0, min_iters=2 if big else 5,
                                             max_iters=3 if big else 40)
        cpu = {"value": it / secs, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"{it} ML-IALM loop iterations of {name} (oracle port of pcp.py:248-296, numpy/OpenBLAS "
                         f"FP64 on the FP32-rounded input), {secs:.1f} s; sigma_1 by an untimed 30-step Lanczos "
                         f"({setup:.1f} s setup)", **host_info()}

    mode = (f"row-sharded x{world} (gloo on one shared device: functional run, NOT a scaling number)" if shared
            else (f"row-sharded x{world}, NCCL all-reduce of the coarse Gram" if world > 1 else "1 GPU"))
    line = {
        "metric": metric_for(name, cfg), "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32" if cfg["dtype"] == "float32" else "f64",
        "data": f"synthetic (seeded generator with BASELINE {name} shapes/distributions)",
        "config": {"workload": workload_for(name, cfg), "seed": args.seed, "step": "one full solve to tolerance "
                   "(sigma_1 Lanczos init + loop) through ml_ialm_solve", "iterations_per_solve": iters / args.steps,
                   "final_gap": hist[-1].feasibility_gap, "final_rank": hist[-1].rank_l,
                   "l2": "256 MB buffer written before every timed step", "parallelism": mode,
                   "shared_device": shared},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": e2e_ms / args.steps, "api": "ml_ialm_solve(pinned torch CPU tensor) -> host L, S, Y"},
        "roofline": roof,
        "kernels": rl,
        "phase_ms_per_iter": per_iter,
        "dominant_phase": dominant,
        "jacobi_sweeps_per_iteration": sweeps_all,
        "lanczos_steps": sink[0].get("lanczos_steps") if sink else None,
        "time_to_tol_ms": total_ms / args.steps,
        "loop_iterations_per_s": (iters / args.steps) / ((total_ms / args.steps - phase_ms.get("lanczos", 0.0)) / 1e3),
        "cpu_baseline": cpu,
        "secondary": secondary or None,
        "gpu_launches": int(launches * args.steps) if launches is not None else None,
        "gpu_launches_per_solve": launches,
        "foreign_kernels": foreign,
        "clocks": clk.summary(),
    }
    return line


def spawn(args):
    """--gpus N without torchrun: launch the N ranks ourselves."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="C5")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the C2 / C3 / C4 side measurements")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3

    from paper_2206_13369_b200.datasets import CONFIGS

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    name = args.config
    cfg = CONFIGS[name]

    if args.impl == "reference":
        if rank == 0:
            run_reference(args, name, cfg)
        return
    if cfg["solver"] != "pcp":
        raise SystemExit("bench.py times an ML-PCP config as the headline (C1, C2 or C5); "
                         "ML-CPCP C3/C4 are reported as secondary keys")
    line = gpu_arm(args, name, cfg, world, rank, local)
    if line is not None:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
