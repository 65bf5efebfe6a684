#!/bin/bash
# round 2: tail thresholds on the HM core (C4 bench, 5+3)
mkdir -p gpurun_out
run() { env "$@" timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/r2t.json; python -c "import json; d=json.load(open('gpurun_out/r2t.json')); t=d['timings_s']; print('$*', round(d['value']/1e6,2), round(t['lookup_active_s'],4), round(t['advance'],3), round(t['collision'],3), round(t['sort'],3))"; }
run EMC_TAIL_N=262144
run EMC_TAIL_N=131072
run EMC_TAIL_N=65536
run EMC_TAIL_N=524288
run EMC_TAIL_N=262144 EMC_TAIL_SUB_N=262144
run EMC_TAIL_N=262144 EMC_TAIL_WARP_N=65536
run EMC_TAIL_N=262144 EMC_TAIL_K=32
