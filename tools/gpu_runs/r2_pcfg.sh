#!/bin/bash
# round 2: CTA shape / register budget of the pipelined lookup (EMC_LK_PCFG), C4 bench each (1 repeated for noise)
mkdir -p gpurun_out
for pc in ${PCS:-1 3 4 5 1}; do
  EMC_LK_PCFG=$pc timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/r2g_bench_$pc.json
  python -c "import json; d=json.load(open('gpurun_out/r2g_bench_$pc.json')); t=d['timings_s']; print($pc, round(d['value']/1e6,2), round(t['lookup_active_s'],4), round(t['advance'],3), round(t['collision'],3))"
done
