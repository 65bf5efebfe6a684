#!/bin/bash
# round 2: C5 / C1 check of the current build against the r2h build and the narrow-P3 variant
mkdir -p gpurun_out
VARS="r2h p3n" WLS="c5 c1" bash tools/gpu_runs/r2_var2.sh
VARS="r2h" WLS="c5" bash tools/gpu_runs/r2_var2.sh
