#!/bin/bash
# round 2: one-compare checkpoint predicate in the lookup's stage loop (base) vs the previous form
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_extensions.py -m gpu -x -q 2>&1 | tail -2
VARS="oldck" WLS="c4 c3" bash tools/gpu_runs/r2_var2.sh
VARS="oldck" WLS="c4" bash tools/gpu_runs/r2_var2.sh
