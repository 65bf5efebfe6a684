timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
for nb in 1 16 64 256; do
EMC_SORT_BANDS=$nb timeout 600 python bench.py --steps 2 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['timings_s']; print('bands=$nb', round(d['value']/1e6,2), 'M/s lookup_act', round(t['lookup_active_s'],3), 'sort', round(t['sort'],3))"
done
