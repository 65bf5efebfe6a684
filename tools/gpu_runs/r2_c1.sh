#!/bin/bash
# round 2: C1 executor timing split + bench line
mkdir -p gpurun_out
timeout 300 python tools/c1_profile.py > gpurun_out/r2_c1.log 2>&1
EMC_TRACE=1 timeout 300 python bench.py --workload c1 --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/r2_c1_trace.log 2>&1
cat gpurun_out/r2_c1.log; grep -c emc-trace gpurun_out/r2_c1_trace.log; tail -1 gpurun_out/r2_c1_trace.log | cut -c1-300
