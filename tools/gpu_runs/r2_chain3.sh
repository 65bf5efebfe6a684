#!/bin/bash
# round 2: chain length 3 with the minimum chaining lanes per warp (1 = ch3, 4, 8), and 6 segments at 8 lanes
mkdir -p gpurun_out
VARS="ch3 ch3m4 ch3m8 ch6m8" WLS="c4 c3 c2" bash tools/gpu_runs/r2_var2.sh
