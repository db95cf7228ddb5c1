#!/bin/bash
# Round-5 (session 4 of build round 2) evidence: GPU tests, smoke, bench (both
# arms), the C5 launch list and ncu --set full of the kernels changed this
# session (one-pass Lanczos with the alternating FP32->FP64 conversion, the
# tridiagonal reduction with the column exchange).
set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/r5_gputest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r5_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r5_smoke.log 2>&1
python bench.py > gpurun_out/r5_bench.json 2> gpurun_out/r5_bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r5_bench_ref.json 2> gpurun_out/r5_bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r5_launches_c5.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/r5_ncu_bench.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name regex:"lz_dtdq_long_kernel" --launch-skip 5 \
    --launch-count 1 -o gpurun_out/r5_full_c5_lz -f python tools/gpu/pcp_solve_iters.py C5 2 > gpurun_out/r5_full_lz.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name regex:"trd_reduce_kernel" --launch-skip 0 \
    --launch-count 1 -o gpurun_out/r5_full_c5_trd -f python tools/gpu/pcp_solve_iters.py C5 2 > gpurun_out/r5_full_trd.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name regex:"trd_reduce_kernel" --launch-skip 0 \
    --launch-count 1 -o gpurun_out/r5_full_c2_trd -f python tools/gpu/pcp_solve_iters.py C2 7 > gpurun_out/r5_full_trd_c2.log 2>&1
tail -2 gpurun_out/r5_gputest.log; cat gpurun_out/r5_smoke.log | tail -2; cut -c1-400 gpurun_out/r5_bench.json; cut -c1-300 gpurun_out/r5_bench_ref.json
