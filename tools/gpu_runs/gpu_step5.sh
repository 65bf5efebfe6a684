set -x
for v in v1 v4; do
EMC_LIBRARY=$PWD/paper_2403_12345_b200/libemc_$v.so timeout 600 python bench.py --steps 2 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['roofline']['achieved'], d['timings_s'])"
done
EMC_LIBRARY=$PWD/paper_2403_12345_b200/libemc_simple.so timeout 1200 ncu --set full --cache-control none --clock-control none --import-source on -k regex:"k_lookup|k_advance|k_collision|k_crossing" -c 4 -o gpurun_out/prof_r2 python tools/profile_step.py --particles 40000000 > gpurun_out/prof2.log 2>&1
tail -3 gpurun_out/prof2.log
