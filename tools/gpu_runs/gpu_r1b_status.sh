# r1 (session 2): re-establish state: GPU parity suite, smoke, full bench, launch list
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; lscpu | grep "Model name" >> gpurun_out/nproc.txt
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/pytest_gpu.log; cat gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/bench_s2.json
cut -c1-2500 gpurun_out/bench_s2.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_s2.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_under_ncu_s2.log 2>&1
echo ncu-done $?
