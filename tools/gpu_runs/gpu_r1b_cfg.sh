mkdir -p gpurun_out
for c in 0 1 2; do echo cfg $c; EMC_LK_CFG=$c timeout 300 python tools/lookup_micro.py 40000000 8 2>&1 | tail -1; done
for c in 1 2; do EMC_LK_CFG=$c timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_cfg$c.json
python -c "import json; d=json.load(open('gpurun_out/bench_cfg$c.json')); t=d['timings_s']; print('cfg $c', round(d['value']/1e6,2), 'M/s', {k: round(v,3) for k,v in t.items() if isinstance(v,float)})"; done
