#!/bin/bash
# round 2: collision register bound revisited after the wide accesses (4 = base, 3, 5 CTAs/SM)
mkdir -p gpurun_out
VARS="col3 col5" WLS="c4 c3" bash tools/gpu_runs/r2_var2.sh
