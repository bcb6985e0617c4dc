#!/bin/bash
# knob sweep: splat grid CTAs per SM; job setup min blocks (now beside the side-stream clear)
mkdir -p gpurun_out
for rep in 1 2; do
  for v in b200 sp8 sp32 sp64 sm6 sm10; do
    FHV_LIB=paper_2211_15460_b200/libfhv_$v.so timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/s68_${v}_$rep.jsonl 2> gpurun_out/s68_${v}_$rep.err
  done
done
