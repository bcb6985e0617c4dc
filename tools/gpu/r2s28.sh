#!/bin/bash
# functional check of the N=2 bench path (two ranks sharing the one GPU, gloo)
mkdir -p gpurun_out
FHV_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline --composite allreduce > gpurun_out/s28_n2.jsonl 2> gpurun_out/s28_n2.err
echo "rc=$?" >> gpurun_out/s28_n2.err
