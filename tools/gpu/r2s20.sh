#!/bin/bash
mkdir -p gpurun_out
FHV_FAST_MATH=1 timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/s20_fast.jsonl 2> gpurun_out/s20_fast.err
timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/s20_base.jsonl 2> gpurun_out/s20_base.err
