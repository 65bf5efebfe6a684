for v in A B C; do
  if [ $v = A ]; then L=paper_2403_12345_b200/libemc.so; else L=build_vars/libemc_$v.so; fi
  echo "== $v"; EMC_LIBRARY=$L timeout 200 python tools/lookup_micro.py 8000000 8 9 2>&1 | tail -2
done
for v in A C; do
  if [ $v = A ]; then L=paper_2403_12345_b200/libemc.so; else L=build_vars/libemc_$v.so; fi
  for pp in 1 0; do
  EMC_LIBRARY=$L EMC_LK_PIPED=$pp timeout 300 python bench.py --workload c4 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v piped $pp c4', round(d['value']/1e6,3), {k: round(v,4) for k,v in d['timings_s'].items() if isinstance(v,float)})"
  EMC_LIBRARY=$L EMC_LK_PIPED=$pp timeout 300 python bench.py --workload c3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v piped $pp c3', round(d['value']/1e6,3), {k: round(v,4) for k,v in d['timings_s'].items() if isinstance(v,float)})"
  done
done
