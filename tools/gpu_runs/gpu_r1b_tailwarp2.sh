run() { env $1 timeout 300 python bench.py --workload $2 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2', round(d['value']/1e6,3), {k: round(v,4) for k,v in d['timings_s'].items() if k in ('lookup',)})"; }
for w in c4 c2 c3; do
for t in 8192 16384 65536 32768; do run EMC_TAIL_WARP_N=$t $w; done
done
