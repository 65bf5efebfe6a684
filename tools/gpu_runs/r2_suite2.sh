#!/bin/bash
# round 2: full GPU suite + driver-shaped bench (HM core default) + reference arm
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2s2_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2s2_pytest.log
tail -4 gpurun_out/r2s2_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/r2s2_bench.json
timeout 900 python bench.py --impl reference 2>&1 | tail -1 > gpurun_out/r2s2_bench_ref.json
for f in r2s2_bench r2s2_bench_ref; do python -c "import json; d=json.load(open('gpurun_out/$f.json')); print('$f', d['value'], d.get('e2e',{}).get('value'), d.get('clocks'), (d.get('cpu_baseline') or {}).get('value'))"; done
