#!/bin/bash
# round 2: tail threshold 131072 vs 262144 (default), alternating, C4 and C2
mkdir -p gpurun_out
for rep in 1 2; do
for e in "EMC_TAIL_N=262144" "EMC_TAIL_N=131072"; do
  for w in c4 c2; do
    env $e timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-counters 2>&1 | grep '^{' | tail -1 > gpurun_out/r2v.json
    python -c "import json; d=json.load(open('gpurun_out/r2v.json')); t=d['timings_s']; print('$e $w', round(d['value']/1e6,2), round(t['lookup_active_s'],4))"
  done
done
done
