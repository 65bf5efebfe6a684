#!/bin/bash
# round 2: GPU test suite + driver-shaped bench (5 + 20) + bench launch list
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2_smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/r2_bench_N1.log 2>&1
echo "bench rc=$?" >> gpurun_out/r2_bench_N1.log
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2_bench_ref.log 2>&1
tail -3 gpurun_out/r2_pytest_gpu.log gpurun_out/r2_bench_N1.log
