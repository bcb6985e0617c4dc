#!/bin/bash
# splat key / winner clears on the build's side stream
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s58_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s58_pytest.log
for rep in 1 2 3; do
  timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/s58_new_$rep.jsonl 2> gpurun_out/s58_new_$rep.err
done
timeout 600 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s58_c5.jsonl 2> gpurun_out/s58_c5.err
