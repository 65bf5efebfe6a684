timeout 300 compute-sanitizer --tool synccheck --print-limit 10 python tools/lookup_micro.py 3000 9 2>&1 | grep -v "^\s*$" | grep -v "Host Frame" | head -40
EMC_FORCE_DEN=0 timeout 60 python tools/lookup_micro.py 20000 9 2>&1 | tail -2
