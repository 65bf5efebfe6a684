for v in I2 I2b3 I2b4 I4 I4b3; do
EMC_LIBRARY=$PWD/paper_2403_12345_b200/libemc_$v.so timeout 600 python bench.py --steps 2 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['timings_s']; print('$v', round(d['value']/1e6,2), 'M/s lookup_act', round(t['lookup_active_s'],3), 'adv', round(t['advance'],3), 'col', round(t['collision'],3))"
done
