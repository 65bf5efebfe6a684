mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_extensions.py -q -x 2>&1 | tail -5
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 900 python bench.py --workload c2 2>&1 | tail -1 > gpurun_out/bench_c2.json
python -c "import json; d=json.load(open('gpurun_out/bench_c2.json')); t=d['timings_s']; print('c2', round(d['value']/1e6,2), 'M/s', {k: round(v,3) for k,v in t.items() if isinstance(v,float)}, d.get('cpu_baseline',{}).get('value'), d['roofline']['achieved'], d['k_mean'])"
