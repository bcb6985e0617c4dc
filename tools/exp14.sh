mkdir -p gpurun_out
for comp in peer allreduce; do
FHV_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline --composite $comp > gpurun_out/exp14_$comp.jsonl 2> gpurun_out/exp14_$comp.err
done
