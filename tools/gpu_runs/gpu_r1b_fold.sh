EMC_TRACE=1 timeout 300 python bench.py --workload c1 --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | grep "fold_ms" | tail -2
for i in 1 2; do timeout 300 python bench.py --workload c1 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1', round(d['value']/1e6,3), d['ms_per_step'], {k: round(v,4) for k,v in d['timings_s'].items() if isinstance(v,float)})"; done
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
