#!/bin/bash
# round 2: quick parity (fingerprints) + C4 bench (5+3) of the current build, twice
mkdir -p gpurun_out
timeout 300 python tools/pcfg_check.py 2>&1 | grep FP
for r in 1 2; do
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/r2q.json
python -c "import json; d=json.load(open('gpurun_out/r2q.json')); t=d['timings_s']; print(round(d['value']/1e6,2), round(t['lookup_active_s'],4), round(t['advance'],3), round(t['collision'],3), round(t['sort'],3))"
done
