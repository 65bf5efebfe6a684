mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multirank.py -q 2>&1 | tail -3
EMC_FORCE_COLLECTIVES=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 2 --warmup 2 --no-cpu-baseline --particles 4000000 2>&1 | tail -2 | cut -c1-400
