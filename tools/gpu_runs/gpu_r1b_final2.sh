# final code: smoke + bench lines (no ncu)
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/bench_r1s9.json
for w in c1 c2 c3 c5; do timeout 900 python bench.py --workload $w 2>&1 | tail -1 > gpurun_out/bench_${w}_r1s9.json; done
for f in bench_r1s9 bench_c1_r1s9 bench_c2_r1s9 bench_c3_r1s9 bench_c5_r1s9; do python -c "import json; d=json.load(open('gpurun_out/$f.json')); print('$f', round(d['value']/1e6,3), 'M/s', d.get('e2e',{}).get('value'), (d.get('cpu_baseline') or {}).get('value'), d['clocks'])"; done
