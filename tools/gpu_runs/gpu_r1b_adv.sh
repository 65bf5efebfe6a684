for lib in libemc libemc_adv2 libemc_adv4; do
EMC_LIBRARY=$PWD/paper_2403_12345_b200/$lib.so timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['timings_s']; print('$lib', round(d['value']/1e6,2), {k: round(v,3) for k,v in t.items() if isinstance(v,float)})"
done
