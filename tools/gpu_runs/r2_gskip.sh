#!/bin/bash
# round 2: table-based per-particle stream skip (base per batch on the host) vs full log-skip
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_extensions.py tests/test_gpu_multirank.py -m gpu -x -q 2>&1 | tail -2
VARS="nogskip" WLS="c4 c3 c2" bash tools/gpu_runs/r2_var2.sh
VARS="nogskip" WLS="c4" bash tools/gpu_runs/r2_var2.sh
