#!/usr/bin/env python
"""Benchmark: ML-PCP iterations/s on BASELINE config C2 (2000x2000 FP32,
rank 100, 10% corruptions, n_H = 250, tol 1e-6), the configuration the
BASELINE metric is quoted on.

A "step" is one full solve (to tolerance) of the C2 instance.  `value` is
iterations/s with D resident in HBM; `e2e` is the same metric through the
public API with a pinned host matrix in and host L, S, Y out.  Rank r of N
holds rows [r*m/N, (r+1)*m/N) (row sharding, NCCL all-reduce of the coarse
Gram each iteration).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ML-PCP iterations/s (C2: 2000x2000 FP32, n_H=250, tol 1e-6)"
UNIT = "iterations/s"


def _ncu_traffic():
    """dram bytes per launch from the committed ncu --set full capture (profiles/)."""
    p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r02_traffic_c2.json")
    try:
        with open(p) as f:
            return json.load(f)["kernels"]
    except (OSError, ValueError, KeyError):
        return {}


def cpcp_secondary(dev, seed):
    """Side measurements (not the headline metric): ML-CPCP C3 to tolerance and
    C4 for 300 iterations, device-resident input, CUDA events, L2 flushed."""
    import torch

    import paper_2206_13369_b200 as pkg
    from paper_2206_13369_b200.datasets import CONFIGS, make_config
    out = {}
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
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
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st = pkg.ml_fwt_solve(D, om, mk(cap))
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        out[name] = {"workload": f"{name} ML-CPCP {m}x{n}, n_H={c['n_coarse']}, tol {c['tol']}, max_iters {cap}",
                     "iterations": st.iter, "converged": st.converged, "solve_ms": ms,
                     "iterations_per_s": st.iter / (ms / 1e3), "dtype": "f32"}
        del D
    return out


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {"hbm_gbs": 6650.0, "_fallback": True}


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
    # timed region: no process spawn (fork) or NVML round trip in this
    # process while the GPU is being timed
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


def cpu_reference_solve(d32, cfg, threads):
    """The reference algorithm (oracle port of pcp.py:213-309) on the host."""
    from threadpoolctl import threadpool_limits

    from oracle import mlrpca_oracle as O
    with threadpool_limits(limits=threads):
        t0 = time.perf_counter()
        r = O.ml_ialm(d32.astype(np.float64), lam=1 / np.sqrt(cfg["m"]), tol=cfg["tol"], levels=cfg["n_coarse"])
        return r.iter, time.perf_counter() - t0


def run_reference(args, cfg, d32):
    threads = len(os.sched_getaffinity(0))
    for _ in range(args.warmup):
        cpu_reference_solve(d32, cfg, threads)
    iters = 0
    secs = 0.0
    for _ in range(args.steps):
        it, s = cpu_reference_solve(d32, cfg, threads)
        iters += it
        secs += s
    value = iters / secs
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, BASELINE C2 shapes/distributions)",
        "config": {"workload": "C2 ML-PCP 2000x2000 rank 100, 10% sparse, n_H=250, tol 1e-6", "seed": args.seed},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{args.steps} full C2 solves (oracle port of mlrpca.ml_ialm_solve, numpy/"
                                   "OpenBLAS, FP64 on the FP32-rounded input)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the ML-CPCP C3/C4 side measurements")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3

    from paper_2206_13369_b200.datasets import CONFIGS, make_config

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    cfg = CONFIGS[args.config]
    assert cfg["solver"] == "pcp", "bench.py times the ML-PCP workload"

    if args.impl == "reference":
        if rank != 0:
            return
        d32, _ = make_config(args.config, args.seed)
        run_reference(args, cfg, d32)
        return

    import torch
    import torch.distributed as dist

    import paper_2206_13369_b200 as pkg
    from paper_2206_13369_b200 import pcp as pcp_mod

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    d_full, _ = make_config(args.config, args.seed)
    m, n = d_full.shape
    r0, r1 = rank * m // world, (rank + 1) * m // world
    d_host = np.ascontiguousarray(d_full[r0:r1])
    opts = pkg.PcpOptions(lam=1 / np.sqrt(max(m, n)), tol_feasibility=cfg["tol"], levels=cfg["n_coarse"])
    D = torch.from_numpy(d_host).to(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2

    def solve(x):
        if world > 1:
            return pkg.ml_ialm_solve_rows(x, opts, m, None)
        return pkg.ml_ialm_solve(x, opts)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    st = None
    for _ in range(args.warmup):
        st = solve(D)  # as in the timed loop: the previous result stays alive
    # ---- value: D resident in HBM (no per-phase event timers in the timed
    # region: they cost ~8% of a C2 solve)
    barrier()
    total_ms, iters = 0.0, 0
    with ClockSampler(local) as clk:
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
    # ---- per-phase CUDA-event timings (roofline): one more solve, untimed
    sink = []
    pcp_mod.TIMING_SINK = sink
    flush.fill_(1.0)
    solve(D)
    torch.cuda.synchronize()
    pcp_mod.TIMING_SINK = None
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    value = iters / (total_ms / 1e3)

    # ---- e2e: pinned host D in, host L/S/Y out, through the public API
    d_pin = torch.from_numpy(d_host).pin_memory()
    st = None
    for _ in range(max(args.warmup, 3)):
        # same pattern as the timed loop (the previous result stays alive while
        # the next solve runs), so torch's pinned host cache holds both result
        # sets before timing starts instead of growing inside the timed region
        st = solve(d_pin)
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
    t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_ms = float(t.item())
    e2e_value = e2e_iters / (e2e_ms / 1e3)
    bytes_el = d_host.dtype.itemsize
    h2d = int(d_host.size * bytes_el)
    d2h = int(3 * d_host.size * bytes_el)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant phase, from the live event timings
    peaks = _peaks()
    phases = {}
    for s in sink:
        for k, v in s.items():
            if isinstance(v, tuple):
                a = phases.setdefault(k, [0.0, 0])
                a[0] += v[0]
                a[1] += v[1]
    nh = cfg["n_coarse"]
    npad = (nh + 63) // 64 * 64
    b = bytes_el
    # B_iter = b (3 m n + 2 m n_H) -- read D, Y, write Y; A' written/read once
    upd_bytes = b * (3 * m * n + 2 * m * npad)
    traffic = _ncu_traffic()
    phase_ms = {k: v[0] for k, v in phases.items()}
    dominant = max(phase_ms, key=phase_ms.get) if phase_ms else None
    sweeps = [x for s in sink for x in s.get("jac_sweeps", [])]
    mean_sweeps = statistics.mean(sweeps) if sweeps else 1.0
    roof = None
    if dominant == "jacobi":
        # Two-sided block Jacobi on the n_p x n_p coarse Gram (FP64): per sweep the
        # block rotations of B~ (8 n_p^3) and of V (4 n_p^3) -> 12 n_p^3 flops.
        ms, cnt = phases["jacobi"]
        flops = 12.0 * npad ** 3 * mean_sweeps
        fp64_peak = 40.0
        ach = flops / (ms / cnt / 1e3) / 1e12
        t = traffic.get("jacobi2_kernel")
        roof = {"bound": "tensor", "kernel": "jacobi2_kernel<cluster> + j2_vapply_kernel (FP64 two-sided block "
                "Jacobi, 16-CTA cluster; latency-bound: one 32x32 rotation chain per round)",
                "achieved": ach, "peak": fp64_peak, "unit": "TFLOP/s", "frac": ach / fp64_peak,
                "peak_source": "nominal B200 FP64 tensor (FP64 not in MEASURED_PEAKS.json)",
                "traffic": t["dram_bytes_per_launch"] if t else None,
                "algorithmic_flops_per_launch": flops, "mean_sweeps": mean_sweeps,
                "flops_formula": "12 n_p^3 per sweep"}
    upd = phases.get("update")
    streaming = None
    if upd:
        ach = upd_bytes / (upd[0] / upd[1] / 1e3) / 1e9
        t = traffic.get("pcp_update_fast")
        streaming = {"bound": "hbm", "kernel": "pcp_update_fast<3,true,4> (FP32 regular-chain fused prolong/shrink/"
                     "dual/restrict, warp per row)", "achieved": ach, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": ach / peaks["hbm_gbs"], "traffic": t["dram_bytes_per_launch"] if t else None,
                     "algorithmic_bytes_per_launch": upd_bytes, "avg_us": 1e3 * upd[0] / upd[1],
                     "bytes_formula": "b (3 m n + 2 m n_p)"}
        if roof is None:
            roof = streaming
    per_iter = {k: round(v / max(1, sum(s.get("iters", 0) for s in sink)), 4) for k, v in phase_ms.items()}

    cpu = None
    if not args.no_cpu_baseline:
        threads = len(os.sched_getaffinity(0))
        it, secs = cpu_reference_solve(d_full, cfg, threads)
        cpu = {"value": it / secs, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"1 full C2 solve ({it} iterations, oracle port of mlrpca.ml_ialm_solve, numpy/OpenBLAS FP64)"}

    lz = statistics.mean(s.get("lanczos_steps", 0) for s in sink) if sink else 0
    # launches per solve (counted in profiles/r02_bench_launches_c2.csv): 21 per loop
    # call (gram 3, pre 6 incl. split-K sums, rank-0 test 1, jacobi + V update 2, after/weights 2,
    # post 4, recon 1, update 1, finalize 1), 3 per Lanczos step (D^T D q, slice sum,
    # update), 11 fixed.  Calls and steps are issued in batches of 4 and the polling
    # is pipelined one batch deep, so one batch of each runs (as no-ops) past the end.
    calls = 4 * math.ceil((iters / args.steps) / 4) + 4
    if world == 1 and n <= 4096:
        lz_launches = 2  # init + the single cooperative Lanczos kernel
    else:
        lz_launches = 3 * (4 * math.ceil(lz / 4) + 4)
    per_solve_launches = 21 * calls + lz_launches + 11
    secondary = cpcp_secondary(dev, args.seed) if (world == 1 and not args.no_secondary) else None
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded generator with BASELINE C2 shapes/distributions)",
        "config": {"workload": "C2 ML-PCP 2000x2000 rank 100, 10% sparse U[-1,1], n_H=250, tol 1e-6",
                   "seed": args.seed, "iterations_per_solve": iters / args.steps,
                   "l2": "256 MB buffer written before every timed step",
                   "parallelism": f"row-sharded x{world}" if world > 1 else "1 GPU"},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": e2e_ms / args.steps},
        "roofline": roof,
        "streaming_kernel": streaming,
        "phase_ms_per_iter": per_iter,
        "dominant_phase": dominant,
        "time_to_tol_ms": total_ms / args.steps,
        "cpu_baseline": cpu,
        "cpcp_configs": secondary,
        "gpu_launches": int(per_solve_launches * args.steps),
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
