for lib in libemc libemc_pf; do
for lb in 256 1024; do
EMC_LIBRARY=$PWD/paper_2403_12345_b200/$lib.so EMC_LOOKUP_BLOCK=$lb timeout 600 python bench.py --steps 2 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['timings_s']; print('$lib lb=$lb', round(d['value']/1e6,2), 'M/s lookup_act', round(t['lookup_active_s'],3), d['k_mean'])"
done
done
