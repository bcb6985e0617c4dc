#!/bin/bash
# N = 2 bench path (two ranks sharing the one GPU over gloo), C3 defaults, short
mkdir -p gpurun_out
FHV_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/s81_n2.jsonl 2> gpurun_out/s81_n2.err; echo "rc=$?" >> gpurun_out/s81_n2.err
FHV_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/s81_ref_n2.jsonl 2> gpurun_out/s81_ref_n2.err; echo "rc=$?" >> gpurun_out/s81_ref_n2.err
