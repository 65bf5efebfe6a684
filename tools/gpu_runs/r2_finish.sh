#!/bin/bash
# round 2: small-population finish kernel: GPU suite, C1 split, C4/C2/C5 with finish thresholds
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r2h_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2h_pytest.log
tail -3 gpurun_out/r2h_pytest.log
timeout 300 python tools/c1_profile.py 2>&1
for f in 0 2048 16384; do
  EMC_FINISH_N=$f timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/r2h_c4_$f.json
  python -c "import json; d=json.load(open('gpurun_out/r2h_c4_$f.json')); t=d['timings_s']; print('c4 finish', $f, round(d['value']/1e6,2), round(t['lookup_active_s'],4), round(t['advance'],3), round(t['collision'],3))"
done
for w in c1 c5 c2; do
  timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/r2h_$w.json
  python -c "import json; d=json.load(open('gpurun_out/r2h_$w.json')); print('$w', round(d['value']/1e6,3))"
done
