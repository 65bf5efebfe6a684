for v in A M1; do
  if [ $v = A ]; then L=paper_2403_12345_b200/libemc.so; else L=build_vars/libemc_m1.so; fi
  for w in c4 c2 c3; do
  EMC_LIBRARY=$L timeout 300 python bench.py --workload $w --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $w', round(d['value']/1e6,3), {k: round(v,4) for k,v in d['timings_s'].items() if isinstance(v,float)})"
  done
done
EMC_LIBRARY=build_vars/libemc_m1.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
