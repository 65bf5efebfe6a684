for w in c4 c3; do
timeout 600 python bench.py --workload $w --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', round(d['value']/1e6,3), round(d['ms_per_step'],2), d['steps']+d['warmup'], {k: round(v,4) for k,v in d['timings_s'].items() if isinstance(v,float)}, d['roofline']['frac'])"
done
EMC_TRACE=1 timeout 600 python bench.py --workload c3 --steps 1 --warmup 3 --no-cpu-baseline 2>&1 | grep emc-trace | awk '{print $2}' | sort | uniq -c
EMC_TRACE=1 timeout 600 python bench.py --workload c3 --steps 1 --warmup 3 --no-cpu-baseline 2>&1 | grep "emc-trace iter" | tail -80 | head -80
