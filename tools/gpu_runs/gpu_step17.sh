timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
timeout 600 python tools/lookup_micro.py 8000000 4 6
timeout 600 python bench.py --steps 2 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['timings_s']; print(round(d['value']/1e6,2), 'M/s', {k: round(v,3) for k,v in t.items() if isinstance(v,float)})"
