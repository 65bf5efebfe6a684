#!/bin/bash
# round 2: GPU suite incl. scale-parity + thread-rank tests; lookup counters; full ncu of one piped lookup launch
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r2s_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2s_pytest_gpu.log
( time timeout 900 python tools/lookup_counters.py --out gpurun_out/r2_lookup_counters.json ) > gpurun_out/r2s_counters.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lookup_piped -s 6 -c 1 -o gpurun_out/r2s_lookup python tools/profile_step.py --particles 40000000 > gpurun_out/r2s_ncu.log 2>&1
echo done
