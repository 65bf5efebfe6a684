#!/bin/bash
# round 2: particles-per-lane variants of the pipelined lookup: parity (fingerprints) + C4 bench per config
mkdir -p gpurun_out
for pc in 1 3 4 5; do
  EMC_LK_PCFG=$pc timeout 300 python tools/pcfg_check.py 2>&1 | grep FP
done > gpurun_out/r2p_fp.log
for pc in 1 3 4 5; do
  EMC_LK_PCFG=$pc timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/r2p_bench_$pc.json
  python -c "import json; d=json.load(open('gpurun_out/r2p_bench_$pc.json')); print($pc, d['value']/1e6, d['timings_s'])"
done > gpurun_out/r2p_bench.log 2>&1
cat gpurun_out/r2p_fp.log gpurun_out/r2p_bench.log
