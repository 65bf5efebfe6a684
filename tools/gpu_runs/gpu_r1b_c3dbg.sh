timeout 600 python bench.py --workload c3 --no-cpu-baseline --steps 2 --warmup 2 2>&1 | tail -5
