#!/bin/bash
# round 2: finish threshold across workloads
mkdir -p gpurun_out
for w in c4 c3 c2 c4pin; do for f in -1 131072 0; do
  if [ $f = -1 ]; then unset EMC_FINISH_N; else export EMC_FINISH_N=$f; fi
  timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-counters 2>&1 | grep '^{' | tail -1 > gpurun_out/r2w.json
  python -c "import json; d=json.load(open('gpurun_out/r2w.json')); t=d['timings_s']; print('$w finish $f', round(d['value']/1e6,2), round(t['lookup_active_s'],4), round(t['advance'],3), round(t['collision'],3))"
done; done
