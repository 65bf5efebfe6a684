mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -x 2>&1 | tail -5
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:k_lookup_staged --csv --log-file gpurun_out/lookup_traffic_r1s2.csv python tools/profile_step.py --particles 40000000 > gpurun_out/lookup_traffic_r1s2.log 2>&1
echo traffic $?
