#!/bin/bash
# ncu --set full of one live launch of the one-pass Lanczos kernel (C5) with
# source-level counters; raw page dumped to CSV.
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on --kernel-name regex:"lz_dtdq_long_kernel" --launch-skip 5 \
    --launch-count 1 -o gpurun_out/s4_lz -f python tools/gpu/pcp_solve_iters.py C5 2 > gpurun_out/s4_lz.log 2>&1
ncu -i gpurun_out/s4_lz.ncu-rep --page raw --csv > gpurun_out/s4_lz_raw.csv 2>/dev/null
ncu -i gpurun_out/s4_lz.ncu-rep --page source --csv > gpurun_out/s4_lz_source.csv 2>/dev/null
tail -3 gpurun_out/s4_lz.log
