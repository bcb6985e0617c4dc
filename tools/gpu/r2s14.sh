#!/bin/bash
mkdir -p gpurun_out
timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/s14_base.jsonl 2> gpurun_out/s14_base.err
FHV_LIB=paper_2211_15460_b200/libfhv_nored.so timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/s14_nored.jsonl 2> gpurun_out/s14_nored.err
