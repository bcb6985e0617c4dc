#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --config C5 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/s44_c5.jsonl 2> gpurun_out/s44_c5.err
