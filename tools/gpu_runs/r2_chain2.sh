#!/bin/bash
# round 2: same-material chain length re-measured after the chain score accumulation (2 = base, 3, 4)
mkdir -p gpurun_out
VARS="ch3 ch4" WLS="c4 c3 c2" bash tools/gpu_runs/r2_var2.sh
