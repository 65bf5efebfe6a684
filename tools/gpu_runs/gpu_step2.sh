set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q 2>&1 | tail -15
timeout 600 python bench.py --particles 4000000 --steps 2 --warmup 2 --no-cpu-baseline 2>&1 | tail -5
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline 2>&1 | tail -5
