for v in w3 w2 w3b3; do
for hb in 0 1; do
EMC_HASH_EXTRA_BITS=$hb EMC_LIBRARY=$PWD/paper_2403_12345_b200/libemc_$v.so timeout 600 python bench.py --steps 2 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['timings_s']; print('$v hb=$hb', round(d['value']/1e6,2), 'M/s lookup_act', round(t['lookup_active_s'],3))"
done
done
