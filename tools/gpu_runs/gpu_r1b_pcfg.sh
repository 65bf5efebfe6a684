run() { EMC_LIBRARY=$1 EMC_LK_PCFG=$2 timeout 300 python bench.py --workload $3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 pcfg $2 $3', round(d['value']/1e6,3), {k: round(v,4) for k,v in d['timings_s'].items() if isinstance(v,float) and k in ('lookup','lookup_active_s')})"; }
for w in c4 c3; do
run paper_2403_12345_b200/libemc.so 0 $w
run build_vars/libemc_d4.so 0 $w
run build_vars/libemc_d4.so 1 $w
run build_vars/libemc_d3.so 1 $w
done
