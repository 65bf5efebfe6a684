#!/bin/bash
# round 2: ncu of k_advance / k_collision on the HM core + launch list of a bench step
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_advance|k_collision" -s 20 -c 2 -o gpurun_out/r2a_advcol python tools/profile_step.py --particles 40000000 > gpurun_out/r2a_ncu.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2a_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-counters > /dev/null 2>&1
echo done
