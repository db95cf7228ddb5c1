#!/bin/bash
# A/B switches (round 3): Gram K-slices on the CPCP configs, Lanczos reorthogonalisation passes on C5
OUT=${OUT:-gpurun_out/r3_ab.log}
for s in default 16 37 74; do
  echo "== MLR_GRAM_SPLITS=$s" >> $OUT
  if [ $s = default ]; then timeout 300 python tools/gpu/cpcp_phase_timing.py >> $OUT 2>&1
  else MLR_GRAM_SPLITS=$s timeout 300 python tools/gpu/cpcp_phase_timing.py >> $OUT 2>&1; fi
done
for r in 0 1; do
  echo "== MLR_LZ_CL_REORTH=$r" >> $OUT
  MLR_LZ_CL_REORTH=$r timeout 300 python tools/gpu/pcp_phase_timing.py C5 >> $OUT 2>&1
done
