#!/bin/bash
# round 2: one-round-trip queue pushes (advance) and claims (collision) vs separate atomics
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_extensions.py -m gpu -x -q 2>&1 | tail -2
VARS="nopush" WLS="c4 c3 c2" bash tools/gpu_runs/r2_var2.sh
VARS="nopush" WLS="c4" bash tools/gpu_runs/r2_var2.sh
