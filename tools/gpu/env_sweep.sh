#!/bin/bash
# Jacobi / coarse-product switches on a config (default C5): one phase-timing
# solve per setting (tools/gpu/pcp_phase_timing.py), results appended to $OUT.
CFG=${CFG:-C5}
OUT=${OUT:-gpurun_out/env_sweep.log}
run() { echo "== $*" >> $OUT; env "$@" timeout 300 python tools/gpu/pcp_phase_timing.py $CFG >> $OUT 2>&1; }
run X=default
run MLR_VA_ROWS=8
run MLR_J2_PER_SM=1
run MLR_J2_DFLOW=2
run MLR_J2_DFLOW=0
run MLR_COARSE_KSPLIT=1
run MLR_COARSE_KSPLIT=4
