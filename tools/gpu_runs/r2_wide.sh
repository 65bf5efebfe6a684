#!/bin/bash
# round 2: 256-bit loads of composition entries and sin/cos table rows, 128-bit log table rows (base) vs before
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_extensions.py -m gpu -x -q 2>&1 | tail -2
VARS="prewide" WLS="c4 c3 c2" bash tools/gpu_runs/r2_var2.sh
VARS="prewide" WLS="c4" bash tools/gpu_runs/r2_var2.sh
