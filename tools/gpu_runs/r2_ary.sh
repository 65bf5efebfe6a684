#!/bin/bash
# round 2: k-ary checkpoint search in collision nuclide selection (ary8 base) vs binary / 4 / 16, COL_MINB=3;
# parity fingerprints first
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
VARS="ary1 ary4 ary16 col3" bash tools/gpu_runs/r2_var2.sh
VARS="ary1" WLS="c4" bash tools/gpu_runs/r2_var2.sh
