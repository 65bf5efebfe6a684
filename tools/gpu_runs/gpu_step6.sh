set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -3
for v in libemc libemc_simple libemc_v5; do
EMC_LIBRARY=$PWD/paper_2403_12345_b200/$v.so timeout 600 python bench.py --steps 2 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['roofline']['achieved'], d['timings_s'])"
done
