#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) or
the raw page of a --set full report into a markdown table for profiles/."""

import collections
import csv
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, out = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            v = float(d["Metric Value"].replace(",", ""))
            unit = d["Metric Unit"]
            ns = v * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(unit, 1)
            out.append((d["Kernel Name"], ns))
    return out


def launch_table(path, title):
    agg = collections.OrderedDict()
    for name, ns in launches(path):
        short = name.split("(")[0].replace("void ", "")
        a = agg.setdefault(short, [0, 0.0])
        a[0] += 1
        a[1] += ns
    tot = sum(v[1] for v in agg.values())
    lines = [f"# {title}", "", f"source: `{path}` (ncu --metrics gpu__time_duration.sum --clock-control none;"
             " cold-cache, serialised launches — compare shares, not absolutes)", "",
             "| kernel | launches | total ms | share | avg us |", "|---|---:|---:|---:|---:|"]
    for k, (n, ns) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{k}` | {n} | {ns / 1e6:.3f} | {100 * ns / tot:.1f}% | {ns / n / 1e3:.2f} |")
    lines.append(f"| **total** | {sum(v[0] for v in agg.values())} | {tot / 1e6:.3f} | 100% | |")
    return "\n".join(lines) + "\n"


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
           "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg",
           "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
           "sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
           "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
           "sm__ops_path_tensor_op_utchmma_src_tf32_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
           "launch__grid_size", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "smsp__issue_active.avg.pct_of_peak_sustained_active"]


def full_table(rep, title):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    lines = [f"## {title}", "", f"source: `{rep}` (ncu --set full --clock-control none)", ""]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        lines.append(f"### `{d.get('Kernel Name', '?').split('(')[0]}` grid {d.get('Grid Size')} block {d.get('Block Size')}")
        lines.append("")
        lines.append("| metric | value |")
        lines.append("|---|---|")
        for m in METRICS:
            if m in d:
                lines.append(f"| {m} | {d[m]} {u.get(m, '')} |")
        lines.append("")
    return "\n".join(lines) + "\n"


if __name__ == "__main__":
    mode, title, paths = sys.argv[1], sys.argv[2], sys.argv[3:]
    if mode == "launches":
        print(launch_table(paths[0], title))
    else:
        print(f"# {title}\n")
        for p in paths:
            print(full_table(p, p.rsplit("/", 1)[-1]))
