for i in 1 2; do timeout 300 python bench.py --workload c5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5', round(d['value']/1e6,3), round(d['ms_per_step'],2), {k: round(v,4) for k,v in d['timings_s'].items() if isinstance(v,float)})"; done
timeout 900 python -m pytest tests/test_gpu_extensions.py -q -x 2>&1 | tail -2
