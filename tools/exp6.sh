mkdir -p gpurun_out
STAGES="pytest bench" bash tools/gpu_round.sh r01s9
timeout 300 python tools/host_profile.py 30 > gpurun_out/r01s9_hostprof.txt 2>&1
timeout 600 python bench.py --config C2 --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/r01s9_C2.jsonl 2> gpurun_out/r01s9_C2.err
