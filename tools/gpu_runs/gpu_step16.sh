timeout 600 python tools/lookup_micro.py 8000000 0 2 4 5 6 7
