#!/bin/bash
# A/B of library builds on one box: gpurun_ab/libA.so (previous) vs the in-tree build.
# usage: bash tools/gpu/s4_ab.sh "C2 C5" [pytest -k expression]
cfgs=${1:-"C2 C5"}
for r in 1 2; do
  for lib in gpurun_ab/libA.so paper_2206_13369_b200/libmlr_b200.so; do
    echo "LIB $lib"
    MLR_LIB_PATH=$PWD/$lib timeout 300 python tools/gpu/pcp_phase_timing.py $cfgs 2>&1 | grep -o "^C[0-9]\|iters [0-9]*\|solve ms [0-9.]*\|'jacobi': ([0-9.]*\|'lanczos': ([0-9.]*\|'gram': ([0-9.]*"
  done
done
if [ -n "$2" ]; then python -m pytest tests -m gpu -x -q -k "$2" 2>&1 | tail -3; fi
