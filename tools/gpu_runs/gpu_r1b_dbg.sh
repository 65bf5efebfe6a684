timeout 120 python tools/lookup_micro.py 20000 8 9 2>&1 | tail -5
EMC_LK_PIPED=1 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -15
