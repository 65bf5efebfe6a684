# ncu --set full of the staged and plain lookup kernels (lookup microbenchmark, 8M particles)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_lookup_staged" -s 1 -c 1 -o gpurun_out/prof_staged python tools/lookup_micro.py 8000000 8 > gpurun_out/prof_staged.log 2>&1
echo staged $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_lookup_bench" -s 1 -c 1 -o gpurun_out/prof_plain python tools/lookup_micro.py 8000000 4 > gpurun_out/prof_plain.log 2>&1
echo plain $?
