EMC_LK_CFG=3 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_extensions.py -q -x 2>&1 | tail -1
for c in 0 3; do
EMC_LK_CFG=$c timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['timings_s']; print('cfg $c', round(d['value']/1e6,2), {k: round(v,3) for k,v in t.items() if isinstance(v,float)})"
done
