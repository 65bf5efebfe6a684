for tn in 262144 0 65536 1000000; do
EMC_TAIL_N=$tn timeout 300 python bench.py --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tail_n $tn', round(d['value']/1e6,3), {k: round(v,4) for k,v in d['timings_s'].items() if isinstance(v,float)})"
done
