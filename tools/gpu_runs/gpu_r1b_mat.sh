run() { env $1 timeout 300 python bench.py --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['value']/1e6,3), {k: round(v,4) for k,v in d['timings_s'].items() if isinstance(v,float)})"; }
run EMC_SORT_MAT=1
run EMC_SORT_MAT=0
run "EMC_SORT_MAT=0 EMC_SORT_FINE=8"
run "EMC_SORT_MAT=0 EMC_SORT_FINE=10"
run EMC_SORT_MAT=1
