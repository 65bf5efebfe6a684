#!/bin/bash
# round 2 experiment: upper bound of removing the advance's tally atomics (results wrong; timing only)
mkdir -p gpurun_out
VARS="noatom" WLS="c4 c3" bash tools/gpu_runs/r2_var2.sh
