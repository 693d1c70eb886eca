#!/bin/bash
# compute-sanitizer evidence for the mbarrier / TMEM / lockstep / last-block
# counter kernels (run on the GPU box): memcheck, racecheck, synccheck and
# initcheck over tools/sanitize_cases.py. Logs land in gpurun_out/sanitize_*.
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck initcheck; do
  mode=""
  [ "$tool" = racecheck ] || [ "$tool" = initcheck ] && mode=quick
  timeout 1500 $CS --tool $tool --print-limit 50 --error-exitcode 9 python tools/sanitize_cases.py $mode \
    > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitize_summary.txt
  tail -3 gpurun_out/sanitize_$tool.log >> gpurun_out/sanitize_summary.txt
done
