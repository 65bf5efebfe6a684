#!/bin/bash
# round 2: full ncu of one pipelined lookup launch (stage fast path build)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lookup_piped -s 6 -c 1 -o gpurun_out/r2n_lookup python tools/profile_step.py --particles 40000000 > gpurun_out/r2n_ncu.log 2>&1
echo done
