for m in nvml smi; do
for w in c1 c4; do
BENCH_CLOCKS=$m timeout 600 python bench.py --workload $w --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$m $w', round(d['value']/1e6,3), round(d['ms_per_step'],2), d['clocks'])"
done; done
