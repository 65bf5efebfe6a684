#!/bin/bash
# round 2: fast-mode k-bin contributions accumulated per thread, one warp reduction per collision launch (base) vs per warp-iteration
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -m gpu -x -q 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_scale_parity.py -m gpu -x -q -k fast_tally 2>&1 | tail -2
VARS="kper" WLS="c4 c3 c2" bash tools/gpu_runs/r2_var2.sh
VARS="kper" WLS="c4" bash tools/gpu_runs/r2_var2.sh
