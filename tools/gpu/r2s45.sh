#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s45_c4.jsonl 2> gpurun_out/s45_c4.err
