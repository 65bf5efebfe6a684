mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_collision" -s 4 -c 1 -o gpurun_out/prof_coll2 python tools/profile_step.py --particles 40000000 > gpurun_out/prof_coll2.log 2>&1
echo prof $?
