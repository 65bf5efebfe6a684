#!/bin/bash
# round 2: butterfly reduce-scatter for fast-mode tally scoring (k_advance);
# fast-mode tests, then base (butterfly) vs all-reduce vs ADV_MINB=2
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "fast or tally or score" 2>&1 | tail -3
VARS="nobfly m2" bash tools/gpu_runs/r2_var2.sh
VARS="nobfly m2" WLS="c4" bash tools/gpu_runs/r2_var2.sh
