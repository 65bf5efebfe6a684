timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
for w in c1 c5 c1 c5 c4 c2; do timeout 300 python bench.py --workload $w --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', round(d['value']/1e6,3), {k: round(v,4) for k,v in d['timings_s'].items() if k in ('advance','collision','lookup','sort')})"; done
