#!/bin/bash
# round 2: re-tune after the event-kernel work: checkpoint stride 8 (build), tail / finish thresholds (env)
mkdir -p gpurun_out
VARS="ck8" WLS="c4 c3" bash tools/gpu_runs/r2_var2.sh
for e in "EMC_TAIL_N=131072" "EMC_TAIL_N=524288" "EMC_FINISH_N=65536" "EMC_FINISH_N=16384"; do
  for w in c4 c3; do
    env $e timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-counters 2>&1 | grep '^{' | tail -1 > gpurun_out/r2v.json
    python -c "import json; d=json.load(open('gpurun_out/r2v.json')); t=d['timings_s']; print('$e $w', round(d['value']/1e6,2), round(t['lookup_active_s'],4), round(t['advance'],3), round(t['collision'],3))"
  done
done
