#!/bin/bash
# round 2: sort-key fine-energy bits re-measured after the event-kernel work (5 = default)
mkdir -p gpurun_out
for e in "EMC_SORT_FINE=5" "EMC_SORT_FINE=4" "EMC_SORT_FINE=6" "EMC_SORT_FINE=3"; do
  for w in c4 c3; do
    env $e timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-counters 2>&1 | grep '^{' | tail -1 > gpurun_out/r2v.json
    python -c "import json; d=json.load(open('gpurun_out/r2v.json')); t=d['timings_s']; print('$e $w', round(d['value']/1e6,2), round(t['lookup_active_s'],4), round(t['sort'],3))"
  done
done
