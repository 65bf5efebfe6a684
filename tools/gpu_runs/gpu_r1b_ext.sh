mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_extensions.py -q -x 2>&1 | tail -15
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
