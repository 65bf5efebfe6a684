timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
for i in 1 2; do
for w in c4 c3; do
timeout 300 python bench.py --workload $w --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', round(d['value']/1e6,3), {k: round(v,4) for k,v in d['timings_s'].items() if isinstance(v,float)})"
done; done
