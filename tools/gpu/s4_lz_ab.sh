#!/bin/bash
# A/B of the FP32 -> FP64 conversion variants of the one-pass Lanczos kernel
# (MLR_LZ_CVT 0: F2F only, 1: alternating F2F / integer, 2: integer only).
mkdir -p gpurun_out
for r in 1 2; do
  for cv in 0 1 2; do
    echo "MLR_LZ_CVT=$cv"
    MLR_LZ_CVT=$cv timeout 200 python tools/gpu/pcp_phase_timing.py C5 2>&1 | grep -o "^C[0-9]\|iters [0-9]*\|solve ms [0-9.]*\|'lanczos': ([0-9.]*\|lanczos steps [0-9]*"
  done
done
MLR_LZ_CVT=1 python -m pytest tests -m gpu -x -q -k "lanczos or c5 or C5" 2>&1 | tail -3
