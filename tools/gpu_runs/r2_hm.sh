#!/bin/bash
# round 2: HM core geometry: parity tests + bench lines (c4hm, c3hm)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_extensions.py -m gpu -q -p no:cacheprovider -k hm_core > gpurun_out/r2m_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2m_pytest.log
tail -3 gpurun_out/r2m_pytest.log
for w in c4hm c3hm; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 2>&1 | tail -1 > gpurun_out/r2m_$w.json
  python -c "import json; d=json.load(open('gpurun_out/r2m_$w.json')); t=d['timings_s']; print('$w', round(d['value']/1e6,3), 'cpu', d.get('cpu_baseline',{}).get('value'), t)"
done
