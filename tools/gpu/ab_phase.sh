# A/B of library builds (MLR_LIB_PATH) on the same box: solve and phase times per solve
# usage: bash tools/gpu/ab_phase.sh libX.so libY.so ... (default: build_trace/libA.so and the in-tree build)
libs="$@"
[ -z "$libs" ] && libs="build_trace/libA.so paper_2206_13369_b200/libmlr_b200.so"
for r in 1 2; do
  for lib in $libs; do
    echo "$lib"; MLR_LIB_PATH=$PWD/$lib timeout 100 python tools/gpu/pcp_phase_timing.py C2 C5 2>&1 | grep -o "^C[0-9]\|solve ms [0-9.]*\|'jacobi': ([0-9.]*\|'lanczos': ([0-9.]*\|lanczos steps [0-9]*"
  done
done
