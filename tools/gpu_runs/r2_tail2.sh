#!/bin/bash
# round 2: tail / finish thresholds after chaining (C4, C3, C2)
mkdir -p gpurun_out
run() { for w in c4 c3 c2; do env "$@" timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-counters 2>&1 | grep '^{' | tail -1 > gpurun_out/r2t.json; python -c "import json; d=json.load(open('gpurun_out/r2t.json')); t=d['timings_s']; print('$* $w', round(d['value']/1e6,2), round(t['lookup_active_s'],4), round(t['advance'],3), round(t['collision'],3), round(t['sort'],3))"; done; }
run EMC_X=default
run EMC_TAIL_N=32768
run EMC_TAIL_N=65536 EMC_FINISH_N=65536
run EMC_FINISH_N=131072
run EMC_TAIL_N=131072 EMC_FINISH_N=131072
