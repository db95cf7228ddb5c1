# trd back-transform columns-per-warp sweep (eigensolve phase per solve)
for cpw in 1 2; do
  echo "cpw $cpw"; MLR_TRD_BACK_CPW=$cpw timeout 100 python tools/gpu/pcp_phase_timing.py C2 C5 2>&1 | grep -o "^C[0-9]\|'jacobi': ([0-9.]*"
done
