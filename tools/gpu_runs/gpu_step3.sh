set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q 2>&1 | tail -3
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_4M.csv python bench.py --particles 4000000 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_lookup|k_advance|k_collision|k_crossing" -c 4 -o gpurun_out/prof_r1 python tools/profile_step.py --particles 4000000 > gpurun_out/prof.log 2>&1
ls -la gpurun_out
