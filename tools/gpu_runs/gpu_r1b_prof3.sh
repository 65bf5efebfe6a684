mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_collision|k_advance|k_crossing|k_sort_keys|Onesweep" -s 40 -c 6 -o gpurun_out/prof_evt python tools/profile_step.py --particles 40000000 > gpurun_out/prof_evt.log 2>&1
echo prof $?
