run() { env $1 timeout 300 python bench.py --workload $2 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2', round(d['value']/1e6,3), {k: round(v,4) for k,v in d['timings_s'].items() if k in ('lookup','advance','collision')})"; }
for w in c4 c3 c2; do
for t in 0 500000 1000000 3000000; do run EMC_SORTED_SUB_N=$t $w; done
done
