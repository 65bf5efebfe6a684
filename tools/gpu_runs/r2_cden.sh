#!/bin/bash
# round 2: constant-memory densities in the pipelined fast path vs shared (EMC_NO_CDEN=1)
mkdir -p gpurun_out
timeout 300 python tools/pcfg_check.py 2>&1 | grep FP > gpurun_out/r2c_fp.log
for v in 0 1; do
  if [ $v = 1 ]; then export EMC_NO_CDEN=1; fi
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/r2c_bench_$v.json
  python -c "import json; d=json.load(open('gpurun_out/r2c_bench_$v.json')); print('nocden=$v', d['value']/1e6, d['timings_s'])" >> gpurun_out/r2c_fp.log
done
cat gpurun_out/r2c_fp.log
