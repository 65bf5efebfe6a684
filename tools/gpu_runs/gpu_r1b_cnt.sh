NB=12 timeout 600 python tools/gpu_runs/c3_seeds.py 2>&1 | tail -4
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
for w in c4; do
timeout 600 python bench.py --workload $w --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', round(d['value']/1e6,3), round(d['ms_per_step'],2), {k: round(v,4) for k,v in d['timings_s'].items() if isinstance(v,float)})"
done
timeout 600 python bench.py --workload c3 --steps 2 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3', round(d['value']/1e6,3), round(d['ms_per_step'],2), {k: round(v,4) for k,v in d['timings_s'].items() if isinstance(v,float)})"
