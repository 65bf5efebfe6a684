#!/bin/bash
# round 2: warp-cooperative finish for staged libraries: parity (fingerprints with finish forced) + C4 thresholds
mkdir -p gpurun_out
EMC_FINISH_N=100000000 timeout 300 python tools/pcfg_check.py 2>&1 | grep FP
EMC_FINISH_N=4096 timeout 300 python tools/pcfg_check.py 2>&1 | grep FP
for f in 0 4096 16384 65536; do
  EMC_FINISH_N=$f timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-counters 2>&1 | grep '^{' | tail -1 > gpurun_out/r2w.json
  python -c "import json; d=json.load(open('gpurun_out/r2w.json')); t=d['timings_s']; print('finish $f', round(d['value']/1e6,2), round(t['lookup_active_s'],4), round(t['advance'],3), round(t['collision'],3), round(t['sort'],3), d['gpu_launches'])"
done
