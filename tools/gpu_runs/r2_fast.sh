#!/bin/bash
# round 2: stage-level fast path of the pipelined lookup: parity fingerprints + C4 bench
mkdir -p gpurun_out
timeout 300 python tools/pcfg_check.py 2>&1 | grep FP > gpurun_out/r2f_fp.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/r2f_bench.json
python -c "import json; d=json.load(open('gpurun_out/r2f_bench.json')); print(d['value']/1e6, d['timings_s'])" >> gpurun_out/r2f_fp.log
cat gpurun_out/r2f_fp.log
