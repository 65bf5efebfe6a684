#!/bin/bash
# round 2: lookup fast-path bracket by double compares instead of 64-bit integer compares
mkdir -p gpurun_out
VARS="hdrf64" WLS="c4 c3" bash tools/gpu_runs/r2_var2.sh
VARS="hdrf64" WLS="c4" bash tools/gpu_runs/r2_var2.sh
