timeout 120 python tools/lookup_micro.py 20000 8 9 2>&1 | tail -2
timeout 200 python tools/lookup_micro.py 8000000 8 9 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
