run() { env $1 timeout 300 python bench.py --workload c5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['value']/1e6,3), round(d['ms_per_step'],2), d['clocks'].get('samples'))"; }
run BENCH_CLOCKS=none
run BENCH_CLOCKS_PERIOD=0.05
run BENCH_CLOCKS_PERIOD=0.5
run BENCH_CLOCKS=none
run BENCH_CLOCKS_PERIOD=0.05
run BENCH_CLOCKS_PERIOD=0.5
