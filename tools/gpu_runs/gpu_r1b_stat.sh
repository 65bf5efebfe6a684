timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k full_size 2>&1 | tail -4
