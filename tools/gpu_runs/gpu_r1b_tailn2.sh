run() { env $1 timeout 300 python bench.py --workload $2 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2', round(d['value']/1e6,3), {k: round(v,4) for k,v in d['timings_s'].items() if k in ('lookup','sort')})"; }
for w in c4 c3 c2; do
for t in 131072 262144 524288; do run EMC_TAIL_N=$t $w; done
done
