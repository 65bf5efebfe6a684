timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
timeout 300 python tools/lookup_micro.py 8000000 8 9 2>&1 | tail -2
for pp in 1 0; do
for w in c4 c3; do
EMC_LK_PIPED=$pp timeout 600 python bench.py --workload $w --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('piped $pp $w', round(d['value']/1e6,3), round(d['ms_per_step'],2), {k: round(v,4) for k,v in d['timings_s'].items() if isinstance(v,float)}, d['k_mean'] if 'k_mean' in d else '')"
done; done
