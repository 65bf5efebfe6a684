#!/bin/bash
# round 2: sort key at 24 bits (fine bits 1: three radix passes) vs 5 fine bits (28 bits, four passes)
mkdir -p gpurun_out
for rep in 1 2; do
for e in "EMC_SORT_FINE=5" "EMC_SORT_FINE=1" "EMC_SORT_FINE=0"; do
  for w in c4; do
    env $e timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-counters 2>&1 | grep '^{' | tail -1 > gpurun_out/r2v.json
    python -c "import json; d=json.load(open('gpurun_out/r2v.json')); t=d['timings_s']; print('$e $w', round(d['value']/1e6,2), round(t['lookup_active_s'],4), round(t['advance'],3), round(t['sort'],3))"
  done
done
done
