#!/bin/bash
# round 2: same-material crossing chains in k_advance: parity subset + benches
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "reference_fingerprint or scale_run or hm_core or tail_lookup or lattice or slab or caps_sort or multirank or edge" > gpurun_out/r2x_pytest.log 2>&1
tail -3 gpurun_out/r2x_pytest.log
for w in c4 c3 c2 c4pin c1 c5; do
  timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-counters 2>&1 | grep '^{' | tail -1 > gpurun_out/r2x.json
  python -c "import json; d=json.load(open('gpurun_out/r2x.json')); t=d['timings_s']; print('$w', round(d['value']/1e6,3), round(t['lookup_active_s'],4), round(t['advance'],3), round(t['collision'],3), round(t['sort'],3), d['gpu_launches'])"
done
