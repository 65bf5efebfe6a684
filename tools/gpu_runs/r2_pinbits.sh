#!/bin/bash
# round 2: lattice pin map as a device bitmask (base) vs int32 per cell
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_extensions.py -m gpu -x -q 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_scale_parity.py -m gpu -x -q -k "c3 and not slow" 2>&1 | tail -2
VARS="pin32" WLS="c4 c3 c2" bash tools/gpu_runs/r2_var2.sh
VARS="pin32" WLS="c4" bash tools/gpu_runs/r2_var2.sh
