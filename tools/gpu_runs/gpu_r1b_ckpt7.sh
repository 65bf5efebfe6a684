# checkpoint 7 (final: + warp-per-particle tail lookup): suite, smoke, benches (c4 + reference, c1, c2, c3, c5), launch list,
# per-kernel ncu, lookup ncu, lookup traffic
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/bench_r1s8.json
timeout 900 python bench.py --impl reference 2>&1 | tail -1 > gpurun_out/bench_ref_r1s8.json
timeout 900 python bench.py --workload c1 2>&1 | tail -1 > gpurun_out/bench_c1_r1s8.json
timeout 900 python bench.py --workload c2 --steps 4 2>&1 | tail -1 > gpurun_out/bench_c2_r1s8.json
timeout 900 python bench.py --workload c3 2>&1 | tail -1 > gpurun_out/bench_c3_r1s8.json
timeout 900 python bench.py --workload c5 2>&1 | tail -1 > gpurun_out/bench_c5_r1s8.json
for f in bench_r1s8 bench_ref_r1s8 bench_c1_r1s8 bench_c2_r1s8 bench_c3_r1s8 bench_c5_r1s8; do python -c "import json; d=json.load(open('gpurun_out/$f.json')); print('$f', round(d['value']/1e6,3), 'M/s', d.get('e2e',{}).get('value'), (d.get('cpu_baseline') or {}).get('value'))"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1s8.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_lookup_piped|k_advance|k_collision|Onesweep" -s 40 -c 7 -o gpurun_out/prof_kernels_r1s8 python tools/profile_step.py --particles 40000000 > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_lookup_piped" -s 6 -c 1 -o gpurun_out/prof_lookup_r1s8 python tools/profile_step.py --particles 40000000 > /dev/null 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:"k_lookup_(piped|staged|warp)" --csv --log-file gpurun_out/lookup_traffic_r1s8.csv python tools/profile_step.py --particles 40000000 > gpurun_out/lookup_traffic_r1s8.log 2>&1
echo done
