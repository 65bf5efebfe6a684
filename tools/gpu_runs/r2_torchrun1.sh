#!/bin/bash
# round 2: the bench's torchrun path (NCCL process group, barrier, max-over-ranks, rank-0 line) forced at world 1
mkdir -p gpurun_out
EMC_FORCE_COLLECTIVES=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline --no-counters 2>&1 | grep '^{' | tail -1 > gpurun_out/r2_torchrun1.json
python -c "import json; d=json.load(open('gpurun_out/r2_torchrun1.json')); print('forced-collective bench', round(d['value']/1e6,2), d['n_gpus'], d.get('scaling'), d['config'].get('parallelism'))"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 1 --steps 3 --warmup 3 2>&1 | grep '^{' | tail -1 | cut -c1-200
