mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
EMC_TAIL_K=3 EMC_TAIL_N=100000000 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fingerprint or staged" 2>&1 | tail -2
for tn in 0 262144 2000000; do
EMC_TAIL_N=$tn timeout 600 python bench.py --workload c2 --steps 3 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['timings_s']; print('c2 tail $tn', round(d['value']/1e6,2), 'M/s', {k: round(v,3) for k,v in t.items() if isinstance(v,float)})"
done
for tn in 0 262144 1000000; do
EMC_TAIL_N=$tn timeout 600 python bench.py --steps 2 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['timings_s']; print('c4 tail $tn', round(d['value']/1e6,2), 'M/s', {k: round(v,3) for k,v in t.items() if isinstance(v,float)})"
done
