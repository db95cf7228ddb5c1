# A/B of two library builds (MLR_LIB_PATH) on the same box: eigensolve phase per solve
for r in 1 2; do
  for lib in build_trace/libA.so paper_2206_13369_b200/libmlr_b200.so; do
    echo "$lib"; MLR_LIB_PATH=$PWD/$lib timeout 100 python tools/gpu/pcp_phase_timing.py C2 C5 2>&1 | grep -o "^C[0-9]\|solve ms [0-9.]*\|'jacobi': ([0-9.]*\|'pre': ([0-9.]*"
  done
done
