mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
EMC_TRACE=1 timeout 600 python tools/profile_step.py --particles 40000000 --batches 3 2> gpurun_out/trace3.txt | tail -1 | cut -c1-100
grep -E "source_init|bank_ms" gpurun_out/trace3.txt
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['timings_s']; print('c4', round(d['value']/1e6,2), {k: round(v,3) for k,v in t.items() if isinstance(v,float)})"
