mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['timings_s']; print('c4', round(d['value']/1e6,2), 'M/s', {k: round(v,3) for k,v in t.items() if isinstance(v,float)})"
timeout 600 python bench.py --workload c2 --steps 3 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2', round(d['value']/1e6,2))"
timeout 600 python bench.py --workload c5 --steps 3 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5', round(d['value']/1e6,2))"
