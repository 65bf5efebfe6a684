mkdir -p gpurun_out
EMC_TRACE=1 timeout 600 python tools/profile_step.py --particles 40000000 --batches 3 2> gpurun_out/trace2.txt | tail -1 | cut -c1-100
grep -E "source_init|bank_ms" gpurun_out/trace2.txt
