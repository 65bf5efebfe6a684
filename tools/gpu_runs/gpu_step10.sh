timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -3
for ro in 1 0; do
EMC_REORDER=$ro timeout 600 python bench.py --steps 2 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['timings_s']; print('reorder=$ro', round(d['value']/1e6,2), 'M/s', {k: round(v,3) for k,v in t.items()})"
done
