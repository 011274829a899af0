#!/bin/bash
# compute-sanitizer evidence: racecheck, synccheck and
# memcheck over tools/sanitize_run.py's workloads.  Logs -> gpurun_out/sanitize/
# Usage on the GPU box: bash tools/sanitize.sh
mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for w in pipeline d512 prim tree; do
    extra=""
    [ "$tool" = "racecheck" ] && extra="--racecheck-report hazard"
    timeout 900 $CS --tool $tool $extra --print-limit 50 --error-exitcode 99 \
      python tools/sanitize_run.py $w > gpurun_out/sanitize/${tool}_${w}.log 2>&1
    echo "$tool $w rc=$?" | tee -a gpurun_out/sanitize/summary.txt
  done
done
