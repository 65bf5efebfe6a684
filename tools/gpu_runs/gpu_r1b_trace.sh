mkdir -p gpurun_out
EMC_TRACE=1 timeout 600 python tools/profile_step.py --particles 40000000 --batches 2 2> gpurun_out/trace.txt | tail -1 | cut -c1-200
grep -c emc-trace gpurun_out/trace.txt
