#!/bin/bash
# round 2: fine energy bits of the lookup sort key (EMC_SORT_FINE) on C4/C3
mkdir -p gpurun_out
for f in 5 3 0 8; do for w in c4 c3; do
  EMC_SORT_FINE=$f timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-counters 2>&1 | grep '^{' | tail -1 > gpurun_out/r2sb.json
  python -c "import json; d=json.load(open('gpurun_out/r2sb.json')); t=d['timings_s']; print('fine $f $w', round(d['value']/1e6,2), round(t['lookup_active_s'],4), round(t['advance'],3), round(t['collision'],3), round(t['sort'],3))"
done; done
