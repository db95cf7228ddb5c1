for sl in 0 50 200 500; do for G in 79 148; do
  echo "sleep $sl G $G"; MLR_TRD_SLEEP=$sl MLR_TRD_G=$G timeout 100 python tools/gpu/pcp_phase_timing.py C5 2>&1 | grep -o "'jacobi': ([0-9.]*"
done; done
for sl in 0 200; do for G in 16 32; do
  echo "C2 sleep $sl G $G"; MLR_TRD_SLEEP=$sl MLR_TRD_G=$G timeout 100 python tools/gpu/pcp_phase_timing.py C2 2>&1 | grep -o "'jacobi': ([0-9.]*"
done; done
