mkdir -p gpurun_out
timeout 300 python tools/lookup_micro.py 40000000 8 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_v5.json
python -c "import json; d=json.load(open('gpurun_out/bench_v5.json')); t=d['timings_s']; print('v5', round(d['value']/1e6,2), 'M/s', {k: round(v,3) for k,v in t.items() if isinstance(v,float)})"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v5.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
echo ncu $?
