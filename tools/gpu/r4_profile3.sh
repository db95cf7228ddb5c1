#!/bin/bash
# Round-4 final: launch list of the C5 bench step and ncu --set full of the
# tridiagonal eigensolver kernels (first live launch) with the final code.
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r4f_launches_c5.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/r4f_ncu_bench.log 2>&1
for K in trd_reduce_kernel trd_bisect_kernel trd_vectors_kernel trd_back_kernel r0_pow_init; do
  ncu --set full --clock-control none --import-source on --kernel-name regex:"$K" --launch-skip 0 --launch-count 1 \
      -o gpurun_out/r4f_full_c5_$K -f python tools/gpu/pcp_solve_iters.py C5 2 > gpurun_out/r4f_full_c5_$K.log 2>&1
done
