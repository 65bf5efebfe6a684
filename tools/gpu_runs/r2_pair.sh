#!/bin/bash
# round 2: two particles per lane in the pipelined lookup (EMC_LK_PCFG 6-9) vs default: parity + C4/C3 bench
mkdir -p gpurun_out
for pc in 1 6 7 8 9; do
  EMC_LK_PCFG=$pc timeout 300 python tools/pcfg_check.py 2>&1 | grep FP | sed "s/^/pcfg $pc /"
  for w in c4 c3; do
    EMC_LK_PCFG=$pc timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-counters 2>&1 | grep '^{' | tail -1 > gpurun_out/r2pp.json
    python -c "import json; d=json.load(open('gpurun_out/r2pp.json')); t=d['timings_s']; print('pcfg $pc $w', round(d['value']/1e6,2), round(t['lookup_active_s'],4), round(t['advance'],3), round(t['collision'],3))"
  done
done
