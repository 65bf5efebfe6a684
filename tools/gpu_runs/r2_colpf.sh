#!/bin/bash
# round 2: L2 prefetch of the next particle line in k_collision
mkdir -p gpurun_out
VARS="nocolpf" WLS="c4 c3" bash tools/gpu_runs/r2_var2.sh
VARS="nocolpf" WLS="c4" bash tools/gpu_runs/r2_var2.sh
