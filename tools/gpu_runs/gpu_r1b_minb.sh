for v in m2_s1 m2_s2 m3_s2 m4_s2 m3_s4 m2_s4; do
EMC_LIBRARY=$PWD/paper_2403_12345_b200/libemc_$v.so timeout 600 python bench.py --steps 2 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['timings_s']; print('$v', round(d['value']/1e6,2), 'M/s', {k: round(v,3) for k,v in t.items() if isinstance(v,float)})"
done
