#!/bin/bash
# Round-4 evidence on the B200 (run from the repo root under gpurun):
#   the default bench (C5 headline + secondaries + CPU baseline), the launch
#   list of the C5 bench step, ncu --set full of the first live launch of the
#   tridiagonal eigensolver kernels at C5.
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/r4_bench.json 2> gpurun_out/r4_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r4_launches_c5.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/r4_ncu_bench.log 2>&1
for K in trd_reduce_kernel trd_bisect_kernel trd_vectors_kernel trd_back_kernel; do
  ncu --set full --clock-control none --import-source on --kernel-name regex:"$K" --launch-skip 0 --launch-count 1 \
      -o gpurun_out/r4_full_c5_$K -f python tools/gpu/pcp_solve_iters.py C5 2 > gpurun_out/r4_full_c5_$K.log 2>&1
done
