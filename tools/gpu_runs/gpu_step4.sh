set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -5
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-2000
EMC_LIBRARY=$PWD/paper_2403_12345_b200/libemc_simple.so timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-2000
