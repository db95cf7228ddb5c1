#!/bin/bash
# Round-3 end-of-session evidence: bench (default args), launch list of a
# C5-only bench, ncu --set full of the one-pass Lanczos and the tcgen05
# reconstruction (live launches), smoke().
mkdir -p gpurun_out
python bench.py > gpurun_out/r3_final_bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3_final_launches_c5.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/r3_final_ncu_bench.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name regex:"lz_dtdq_long_kernel" --launch-skip 3 \
    --launch-count 1 -o gpurun_out/r3_final_lz -f python tools/gpu/pcp_solve_iters.py C5 3 > gpurun_out/r3_final_lz.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3_final_smoke.log 2>&1
