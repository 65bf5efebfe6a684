timeout 120 python tools/lookup_micro.py 20000 9 2>&1 | grep -v "^ " | sort | uniq -c | sort -rn | head -20
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k fresh 2>&1 | grep "emc-dbg\|passed\|failed" | sort | uniq -c | sort -rn | head -20
