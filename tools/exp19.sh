mkdir -p gpurun_out
timeout 600 python bench.py --config C2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/exp19_C2a.jsonl 2>&1
timeout 600 python bench.py --config C2 --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/exp19_C2b.jsonl 2>&1
