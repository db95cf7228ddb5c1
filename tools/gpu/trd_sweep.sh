# trd grid-size sweep on C5 (eigensolve phase per solve)
for G in 79 100 125 148; do
  echo "G $G"; MLR_TRD_G=$G timeout 100 python tools/gpu/pcp_phase_timing.py C5 2>&1 | grep -o "'jacobi': ([0-9.]*"
done
