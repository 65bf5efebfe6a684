for f in 5 0 5 0; do
EMC_SORT_FINE=$f timeout 300 python bench.py --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fine $f', round(d['value']/1e6,3), {k: round(v,4) for k,v in d['timings_s'].items() if isinstance(v,float)})"
done
