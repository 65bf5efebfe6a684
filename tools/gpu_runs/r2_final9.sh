#!/bin/bash
# round 2 final (r2m: + chains of 3): GPU suite, smoke, every workload's bench line (driver shape 5+20), reference arm,
# launch list, ncu of the top kernels, full-batch lookup counters (committed fallback for bench.py)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2m_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2m_pytest.log
tail -3 gpurun_out/r2m_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python tools/lookup_counters.py --out gpurun_out/r2_lookup_counters.json > gpurun_out/r2m_counters.log 2>&1
for w in c4 c4pin c3 c3pin c2 c1 c5; do
  timeout 900 python bench.py --workload $w 2>&1 | grep '^{' | tail -1 > gpurun_out/r2m_bench_$w.json
  python -c "import json; d=json.load(open('gpurun_out/r2m_bench_$w.json')); r=d['roofline']; print('$w', round(d['value']/1e6,3), 'M/s e2e', round(d['e2e']['value']/1e6,3), 'cpu', (d.get('cpu_baseline') or {}).get('value'), 'l1frac', r.get('frac'), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
timeout 900 python bench.py --impl reference 2>&1 | grep '^{' | tail -1 > gpurun_out/r2m_bench_reference.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2m_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-counters > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_lookup_piped|k_advance|k_collision" -s 30 -c 3 -o gpurun_out/r2m_kernels python tools/profile_step.py --particles 40000000 > /dev/null 2>&1
echo done
