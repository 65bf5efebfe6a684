EMC_LK_CFG=3 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "preset251" 2>&1 | grep -E "Error|assert|^E " | head -20
