EMC_TRACE=1 timeout 300 python bench.py --workload c1 --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | grep -E "fold_ms|bank_ms" | tail -4
timeout 600 python bench.py --workload c1 --steps 10 --warmup 10 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1', round(d['value']/1e6,3), d['ms_per_step'], {k: round(v,4) for k,v in d['timings_s'].items() if isinstance(v,float)}, d['gpu_launches'], d['extra'] if 'extra' in d else '')"
timeout 600 python -m pytest tests -q -m gpu -x -k "determin or c1 or golden" 2>&1 | tail -2
