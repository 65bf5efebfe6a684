for w in c3 c4; do
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_lookup_staged --launch-skip 20 --launch-count 1 -o gpurun_out/ncu_lookup_$w python bench.py --workload $w --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_$w.log 2>&1
tail -2 gpurun_out/ncu_$w.log
done
