for lb in 1024 512 256; do
EMC_SORT_BANDS=1 EMC_LOOKUP_BLOCK=$lb timeout 600 python bench.py --steps 2 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['timings_s']; print('lb=$lb', round(d['value']/1e6,2), 'M/s lookup_act', round(t['lookup_active_s'],3))"
done
EMC_SORT_BANDS=64 EMC_LOOKUP_BLOCK=1024 timeout 600 python bench.py --steps 2 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['timings_s']; print('lb=1024 bands64', round(d['value']/1e6,2), 'M/s lookup_act', round(t['lookup_active_s'],3))"
