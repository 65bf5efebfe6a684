timeout 600 python tools/lookup_micro.py 8000000 0 1 2 3
