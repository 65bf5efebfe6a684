run() { EMC_LIBRARY=$1 timeout 300 python bench.py --workload $2 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2', round(d['value']/1e6,3), {k: round(v,4) for k,v in d['timings_s'].items() if k in ('advance','collision','lookup')})"; }
for w in c4 c5; do
run paper_2403_12345_b200/libemc.so $w
for n in adv4 adv2 col5 col3; do run build_vars/libemc_$n.so $w; done
done
