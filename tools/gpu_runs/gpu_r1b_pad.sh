timeout 300 python tools/lookup_micro.py 40000000 8 2>&1 | tail -1
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for r in 1 2; do
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['timings_s']; print('c4', round(d['value']/1e6,2), {k: round(v,3) for k,v in t.items() if isinstance(v,float)})"
done
