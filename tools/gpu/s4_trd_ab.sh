#!/bin/bash
# A/B of the tridiagonal reduction's exchange: MLR_TRD_COLX=0 (owner publishes
# row j + 1 after its update) vs 1 (every row's entry of column j + 1 travels
# with p_i).  Then the eigensolver parity tests with the new default.
for r in 1 2; do
  for cx in 0 1; do
    echo "MLR_TRD_COLX=$cx"
    MLR_TRD_COLX=$cx timeout 300 python tools/gpu/pcp_phase_timing.py C1 C2 C5 2>&1 | grep -o "^C[0-9]\|iters [0-9]*\|solve ms [0-9.]*\|'jacobi': ([0-9.]*"
  done
done
python -m pytest tests -m gpu -x -q -k "eigensolver or trd or tridiag or c1 or c2 or c5 or C5 or determin" 2>&1 | tail -3
