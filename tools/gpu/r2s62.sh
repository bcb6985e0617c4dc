#!/bin/bash
mkdir -p gpurun_out
for k in 20 60; do
  timeout 600 python bench.py --steps $k --warmup 3 --no-cpu-baseline > gpurun_out/s62_k$k.jsonl 2> gpurun_out/s62_k$k.err
done
