#!/bin/bash
# compute-sanitizer over the small cases (only our kernels: regex mlr::);
# summaries -> gpurun_out/r3_sanitize_<tool>.log
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 $CS --tool $tool --kernel-name regex:mlr --error-exitcode 9 --print-limit 20 \
      python tools/gpu/sanitize_cases.py > gpurun_out/r3_sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/r3_sanitize_summary.log
  tail -3 gpurun_out/r3_sanitize_$tool.log >> gpurun_out/r3_sanitize_summary.log
done
