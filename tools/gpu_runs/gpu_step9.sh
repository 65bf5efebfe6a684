mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; lscpu | grep "Model name" >> gpurun_out/nproc.txt
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/bench_r1.json
cat gpurun_out/bench_r1.json | cut -c1-3000
timeout 900 python bench.py --impl reference 2>&1 | tail -1 > gpurun_out/bench_ref_r1.json
cat gpurun_out/bench_ref_r1.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_40M.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_under_ncu40.log 2>&1
timeout 1200 ncu --set full --cache-control none --clock-control none --import-source on -k regex:"k_lookup" -c 1 -o gpurun_out/prof_lookup_r1 python tools/profile_step.py --particles 40000000 > gpurun_out/prof3.log 2>&1
tail -2 gpurun_out/prof3.log
