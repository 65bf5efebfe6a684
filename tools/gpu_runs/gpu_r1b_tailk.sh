run() { env $1 timeout 300 python bench.py --workload $2 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2', round(d['value']/1e6,3), round(d['ms_per_step'],2), d['gpu_launches'])"; }
for w in c1 c5; do
run EMC_TAIL_K=16 $w
run EMC_TAIL_K=32 $w
run EMC_TAIL_K=8 $w
run "EMC_TAIL_K=16 EMC_TAIL_N=65536" $w
run "EMC_TAIL_K=16 EMC_TAIL_N=1000000" $w
done
