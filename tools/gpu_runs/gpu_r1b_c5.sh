mkdir -p gpurun_out
timeout 900 python bench.py --workload c5 2>&1 | tail -1 > gpurun_out/bench_c5.json
python -c "import json; d=json.load(open('gpurun_out/bench_c5.json')); t=d['timings_s']; print('c5', round(d['value']/1e6,2), 'M/s', {k: round(v,3) for k,v in t.items() if isinstance(v,float)}, d.get('mesh'), d.get('cpu_baseline',{}).get('value'))"
timeout 600 python bench.py --workload c5 --impl reference --steps 2 --warmup 1 2>&1 | tail -1 | cut -c1-300
timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4', round(d['value']/1e6,2))"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python bench.py --workload c5 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
echo ncu $?
