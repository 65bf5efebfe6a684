# staged lookup v2 (interval records, stage density blocks, pipelined producer)
mkdir -p gpurun_out
timeout 300 python tools/lookup_micro.py 8000000 4 8 2>&1 | tail -2
timeout 300 python tools/lookup_micro.py 40000000 8 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_staged2.json
python -c "import json; d=json.load(open('gpurun_out/bench_staged2.json')); t=d['timings_s']; print('staged', round(d['value']/1e6,2), 'M/s', {k: round(v,3) for k,v in t.items() if isinstance(v,float)}, d['roofline']['achieved'])"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_lookup_staged" -s 1 -c 1 -o gpurun_out/prof_staged2 python tools/lookup_micro.py 8000000 8 > gpurun_out/prof_staged2.log 2>&1
echo prof $?
