#!/bin/bash
# Round-5 final evidence with the last code: GPU tests, smoke, bench (both
# arms), C5 launch list, ncu --set full of the tridiagonal kernels.
set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/r5c_gputest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r5c_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r5c_smoke.log 2>&1
python bench.py > gpurun_out/r5c_bench.json 2> gpurun_out/r5c_bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r5c_bench_ref.json 2> gpurun_out/r5c_bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r5c_launches_c5.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/r5c_ncu_bench.log 2>&1
for K in trd_reduce_kernel trd_back_kernel; do
  ncu --set full --clock-control none --import-source on --kernel-name regex:"$K" --launch-skip 0 --launch-count 1 \
      -o gpurun_out/r5c_full_c5_$K -f python tools/gpu/pcp_solve_iters.py C5 2 > gpurun_out/r5c_full_c5_$K.log 2>&1
done
ncu --set full --clock-control none --import-source on --kernel-name regex:"trd_reduce_kernel" --launch-skip 0 \
    --launch-count 1 -o gpurun_out/r5c_full_c2_trd -f python tools/gpu/pcp_solve_iters.py C2 7 > gpurun_out/r5c_full_trd_c2.log 2>&1
tail -2 gpurun_out/r5c_gputest.log; tail -2 gpurun_out/r5c_smoke.log; cut -c1-300 gpurun_out/r5c_bench.json
