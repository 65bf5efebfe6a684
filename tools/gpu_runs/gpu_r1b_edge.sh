timeout 900 python -m pytest tests/test_gpu_extensions.py -q -x -k edge 2>&1 | tail -3
