#!/bin/bash
# round 2: control-block counters on separate L2 lines (base) vs packed
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
VARS="packed" WLS="c4 c3 c2" bash tools/gpu_runs/r2_var2.sh
VARS="packed" WLS="c4" bash tools/gpu_runs/r2_var2.sh
