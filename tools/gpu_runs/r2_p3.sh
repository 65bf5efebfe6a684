#!/bin/bash
# round 2: particle bookkeeping sector (P3) as one 256-bit load / store (base) vs struct copies
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_extensions.py tests/test_gpu_multirank.py -m gpu -x -q 2>&1 | tail -2
VARS="p3n" WLS="c4 c3 c2" bash tools/gpu_runs/r2_var2.sh
VARS="p3n" WLS="c4" bash tools/gpu_runs/r2_var2.sh
