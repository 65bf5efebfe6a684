timeout 300 python tools/lookup_micro.py 40000000 8 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_extensions.py -q -x 2>&1 | tail -1
for r in 1 2; do
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['timings_s']; print('c4', round(d['value']/1e6,2), {k: round(v,3) for k,v in t.items() if isinstance(v,float)})"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_lookup_staged" -s 1 -c 1 -o gpurun_out/prof_staged10 python tools/lookup_micro.py 8000000 8 > /dev/null 2>&1
