timeout 600 python bench.py --workload c3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3', round(d['value']/1e6,2), d['k_mean'])"
timeout 600 python bench.py --workload c1 --steps 10 --warmup 10 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1', round(d['value']/1e6,3), d['k_mean'])"
timeout 600 python bench.py --workload c1 --impl reference --steps 10 --warmup 10 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1 ref', round(d['value']/1e6,3))"
timeout 600 python bench.py --workload c3 --impl reference --steps 2 --warmup 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 ref', round(d['value']/1e6,3))"
