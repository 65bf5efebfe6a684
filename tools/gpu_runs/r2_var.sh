#!/bin/bash
# round 2: compile-time variants (register bounds of the event kernels, collision walk width) on the C4 bench
mkdir -p gpurun_out
for v in base ${VARS:-advminb4 colminb3 colminb5 walk2}; do
  if [ $v = base ]; then unset EMC_LIBRARY; else export EMC_LIBRARY=$PWD/build/var/libemc_$v.so; fi
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-counters 2>&1 | grep '^{' | tail -1 > gpurun_out/r2v.json
  python -c "import json; d=json.load(open('gpurun_out/r2v.json')); t=d['timings_s']; print('$v', round(d['value']/1e6,2), round(t['lookup_active_s'],4), round(t['advance'],3), round(t['collision'],3), round(t['sort'],3))"
done
