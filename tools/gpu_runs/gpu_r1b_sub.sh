EMC_TAIL_WARP_N=0 EMC_TAIL_SUB_N=262144 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
EMC_TAIL_WARP_N=4 EMC_TAIL_SUB_N=262144 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fingerprint or fresh" 2>&1 | tail -2
run() { env $1 timeout 300 python bench.py --workload $2 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2', round(d['value']/1e6,3), {k: round(v,4) for k,v in d['timings_s'].items() if k in ('lookup',)})"; }
for w in c4 c2 c3; do
run "EMC_TAIL_SUB_N=0" $w
run "EMC_TAIL_SUB_N=131072" $w
run "EMC_TAIL_SUB_N=262144" $w
done
