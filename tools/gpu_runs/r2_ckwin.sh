#!/bin/bash
# round 2: interpolated first-probe window of the collision's checkpoint search (6 = base) vs binary / 4 / 8
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_extensions.py -m gpu -x -q 2>&1 | tail -2
VARS="win0 win4 win8" WLS="c4 c3" bash tools/gpu_runs/r2_var2.sh
VARS="win0" WLS="c4" bash tools/gpu_runs/r2_var2.sh
