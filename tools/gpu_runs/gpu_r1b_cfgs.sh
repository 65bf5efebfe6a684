for c in 0 1 2 3; do
EMC_LK_CFG=$c timeout 600 python bench.py --workload c3 --steps 2 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 cfg $c', round(d['value']/1e6,3), round(d['ms_per_step'],2), {k: round(v,4) for k,v in d['timings_s'].items() if isinstance(v,float)})"
done
