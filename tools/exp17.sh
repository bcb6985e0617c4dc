mkdir -p gpurun_out
FHV_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29551 bench.py --config C5 --gpus 2 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/exp17_c5x2.jsonl 2> gpurun_out/exp17_c5x2.err
