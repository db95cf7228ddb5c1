#!/bin/bash
# ncu --set full of the round-3 kernels (tcgen05 reconstruction, pipelined
# long-row Lanczos, Gram with the new K-slice count) at C5.
mkdir -p gpurun_out
for K in tc_recon_kernel lz_dtdq_long_kernel gram128_kernel; do
  ncu --set full --clock-control none --import-source on --kernel-name regex:"$K" --launch-skip 2 --launch-count 1 \
      -o gpurun_out/r3_full2_c5_$K -f python tools/gpu/pcp_solve_iters.py C5 12 > gpurun_out/r3_full2_c5_$K.log 2>&1
done
