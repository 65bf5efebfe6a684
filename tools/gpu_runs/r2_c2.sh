#!/bin/bash
# round 2: C2 (1M particles) tail / finish thresholds
mkdir -p gpurun_out
run() { env "$@" timeout 300 python bench.py --workload c2 --steps 10 --warmup 3 --no-cpu-baseline --no-counters 2>&1 | grep '^{' | tail -1 > gpurun_out/r2c2.json; python -c "import json; d=json.load(open('gpurun_out/r2c2.json')); t=d['timings_s']; print('$*', round(d['value']/1e6,2), round(t['lookup_active_s'],4), round(t['advance'],3), round(t['collision'],3), round(t['sort'],3), d['gpu_launches'])"; }
run EMC_X=default
run EMC_TAIL_N=524288
run EMC_TAIL_N=1100000
run EMC_TAIL_N=524288 EMC_TAIL_K=32
run EMC_FINISH_N=65536
run EMC_FINISH_N=16384
