#!/bin/bash
# round 2: compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_run.py
# (EMC_TAIL_N=0: sorted sweeps through the pipelined staged lookup even at 20k particles; default: tail + warp finish)
mkdir -p gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
for env in "EMC_TAIL_N=0" "EMC_TAIL_N=262144"; do
  for tool in memcheck racecheck synccheck; do
    echo "== $tool $env"
    env $env timeout 1500 $S --tool $tool --print-limit 20 python tools/sanitize_run.py 2>&1 | grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Error|error|k \[|slab|history" | head -12
  done
done > gpurun_out/r2_sanitize.txt 2>&1
cat gpurun_out/r2_sanitize.txt
