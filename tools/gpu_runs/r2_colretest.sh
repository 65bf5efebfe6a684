#!/bin/bash
# round 2: collision options re-measured after the 256-bit accesses: isotropic inline, next-line prefetch
mkdir -p gpurun_out
VARS="isoinl colpf" WLS="c4 c3" bash tools/gpu_runs/r2_var2.sh
