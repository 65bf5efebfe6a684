timeout 120 python tools/lookup_micro.py 20000 8 2>&1 | tail -2
timeout 120 python tools/lookup_micro.py 20000 9 2>&1 | grep -v "^ " | tail -4
timeout 400 compute-sanitizer --tool memcheck --print-limit 5 python tools/lookup_micro.py 5000 9 2>&1 | grep -v "^\s*$" | head -40
timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_gpu_parity.py -q -x -k fresh 2>&1 | grep -v "^\s*$" | head -40
