#!/bin/bash
# round 2: driver-shaped bench with the live lookup-counter sample (roofline on the L1TEX data pipe)
mkdir -p gpurun_out
( time timeout 900 python bench.py ) > gpurun_out/r2r_bench.log 2>&1
tail -1 gpurun_out/r2r_bench.json 2>/dev/null
grep '^{' gpurun_out/r2r_bench.log | tail -1 > gpurun_out/r2r_bench.json
python -c "import json; d=json.load(open('gpurun_out/r2r_bench.json')); print(d['value']/1e6, json.dumps(d['roofline'], indent=1))"
tail -4 gpurun_out/r2r_bench.log
