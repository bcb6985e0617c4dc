mkdir -p gpurun_out
STAGES="pytest bench" bash tools/gpu_round.sh r01s8
timeout 600 python bench.py --config C2 --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/r01s8_C2.jsonl 2> gpurun_out/r01s8_C2.err
