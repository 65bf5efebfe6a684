# staged lookup: micro (plain vs staged), parity suite, bench both kernels
mkdir -p gpurun_out
timeout 300 python tools/lookup_micro.py 8000000 4 8 2>&1 | tail -3
timeout 300 python tools/lookup_micro.py 40000000 4 8 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_staged.json
python -c "import json; d=json.load(open('gpurun_out/bench_staged.json')); t=d['timings_s']; print('staged', round(d['value']/1e6,2), 'M/s', {k: round(v,3) for k,v in t.items() if isinstance(v,float)}, d['roofline']['achieved'])"
EMC_LOOKUP=plain timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_plain.json
python -c "import json; d=json.load(open('gpurun_out/bench_plain.json')); t=d['timings_s']; print('plain', round(d['value']/1e6,2), 'M/s', {k: round(v,3) for k,v in t.items() if isinstance(v,float)})"
