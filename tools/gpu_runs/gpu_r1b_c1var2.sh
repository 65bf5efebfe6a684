for i in 1 2 3 4; do timeout 300 python bench.py --workload c1 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1', round(d['value']/1e6,3), round(d['ms_per_step'],2), d['clocks']['samples'])"; done
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
