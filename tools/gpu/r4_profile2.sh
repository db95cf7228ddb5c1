#!/bin/bash
# Round-4: ncu --set full of the FIRST (live) launch at C5 of the 3xTF32
# tcgen05 reconstruction, the DMMA Gram and the fused update pass (tensor-pipe
# and HBM counters the north star asks for), plus C4's CPCP update pass.
set -x
mkdir -p gpurun_out
for K in tc_recon_kernel gram128_kernel pcp_update_fast; do
  ncu --set full --clock-control none --import-source on --kernel-name regex:"$K" --launch-skip 0 --launch-count 1 \
      -o gpurun_out/r4b_full_c5_$K -f python tools/gpu/pcp_solve_iters.py C5 2 > gpurun_out/r4b_full_c5_$K.log 2>&1
done
