#!/bin/bash
# round 2: full ncu of k_advance / k_collision after the wide P3 accesses
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_advance|k_collision" -s 20 -c 2 -o gpurun_out/r2j_advcol python tools/profile_step.py --particles 40000000 > gpurun_out/r2j_ncu.log 2>&1
echo done
