#!/bin/bash
# round 2: compile-time variants on C4 and C3 benches (5+3)
mkdir -p gpurun_out
for v in base ${VARS}; do
  if [ $v = base ]; then unset EMC_LIBRARY; else export EMC_LIBRARY=$PWD/build/var/libemc_$v.so; fi
  for w in ${WLS:-c4 c3}; do
  timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-counters 2>&1 | grep '^{' | tail -1 > gpurun_out/r2v.json
  python -c "import json; d=json.load(open('gpurun_out/r2v.json')); t=d['timings_s']; print('$v $w', round(d['value']/1e6,2), round(t['lookup_active_s'],4), round(t['advance'],3), round(t['collision'],3), round(t['sort'],3))"
  done
done
