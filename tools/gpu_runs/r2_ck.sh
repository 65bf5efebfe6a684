#!/bin/bash
# round 2: sigma_t checkpoint layout (row-major vs particle-major): parity + C4 bench
mkdir -p gpurun_out
for pm in 0 1; do
  EMC_CK_PMAJOR=$pm timeout 300 python tools/pcfg_check.py 2>&1 | grep FP
  EMC_CK_PMAJOR=$pm timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-counters 2>&1 | grep '^{' | tail -1 > gpurun_out/r2k.json
  python -c "import json; d=json.load(open('gpurun_out/r2k.json')); t=d['timings_s']; print('pmajor $pm', round(d['value']/1e6,2), round(t['lookup_active_s'],4), round(t['advance'],3), round(t['collision'],3), round(t['sort'],3))"
done
