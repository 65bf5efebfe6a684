mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_collision|k_advance|k_reorder" -s 30 -c 3 -o gpurun_out/prof_coll python tools/profile_step.py --particles 40000000 > gpurun_out/prof_coll.log 2>&1
echo prof $?
