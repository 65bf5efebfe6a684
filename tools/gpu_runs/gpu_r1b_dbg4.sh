timeout 120 python tools/lookup_micro.py 20000 9 2>&1 | grep "emc" | head -60
