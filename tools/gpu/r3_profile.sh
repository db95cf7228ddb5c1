#!/bin/bash
# Round-3 evidence on the B200 (run from the repo root under gpurun):
#   launch list of the C5 bench (duration only), ncu --set full of the live
#   C5 kernels (first launch of each), compute-sanitizer on small solves.
set -x
mkdir -p gpurun_out
NCU=ncu
# 1. bench launch list (C5 only, one timed step)
$NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3_launches_c5.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/r3_ncu_bench.log 2>&1
# 2. --set full of the first live launch of each C5 kernel (iteration 1 / Lanczos step 0)
for K in pcp_update_fast gram128_kernel lz_dtdq_long_kernel jacobi2_kernel j2_vapply_kernel; do
  $NCU --set full --clock-control none --import-source on --kernel-name regex:"$K" --launch-skip 0 --launch-count 1 \
      -o gpurun_out/r3_full_c5_$K -f python tools/gpu/pcp_solve_iters.py C5 3 > gpurun_out/r3_full_c5_$K.log 2>&1
done
# the reconstruction GEMM (gemm_f64_kernel with M = m rows) is the 4th gemm_f64 launch of iteration 1
$NCU --set full --clock-control none --import-source on --kernel-name regex:"gemm_f64_kernel" --launch-skip 0 \
    --launch-count 8 -o gpurun_out/r3_full_c5_gemm -f python tools/gpu/pcp_solve_iters.py C5 2 > gpurun_out/r3_full_c5_gemm.log 2>&1
