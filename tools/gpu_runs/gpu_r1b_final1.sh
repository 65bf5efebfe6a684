# r1 session 2 checkpoint: parity suite, smoke, full bench (+cpu baseline), reference arm,
# launch list, ncu --set full of the staged lookup (mid-batch launch at C4 40M)
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; lscpu | grep "Model name" >> gpurun_out/nproc.txt
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/bench_r1s2.json
cut -c1-400 gpurun_out/bench_r1s2.json
timeout 900 python bench.py --impl reference 2>&1 | tail -1 > gpurun_out/bench_ref_r1s2.json
cut -c1-300 gpurun_out/bench_ref_r1s2.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1s2.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
echo launches $?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_lookup_staged" -s 6 -c 1 -o gpurun_out/prof_lookup_r1s2 python tools/profile_step.py --particles 40000000 > gpurun_out/prof_lookup_r1s2.log 2>&1
echo prof $?
