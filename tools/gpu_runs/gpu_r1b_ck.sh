timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fingerprint or staged or caps" 2>&1 | tail -1
for rep in 1 2; do
for lib in libemc_base libemc_ck2; do
EMC_LIBRARY=$PWD/paper_2403_12345_b200/$lib.so timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['timings_s']; print('$lib', round(d['value']/1e6,2), {k: round(v,3) for k,v in t.items() if isinstance(v,float)})"
done; done
