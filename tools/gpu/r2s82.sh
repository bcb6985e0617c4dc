#!/bin/bash
# splat index / resolve grids: CTAs per SM
mkdir -p gpurun_out
for rep in 1 2; do
  for v in b200 i24 i32 r8 r32; do
    FHV_LIB=paper_2211_15460_b200/libfhv_$v.so timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/s82_${v}_$rep.jsonl 2> gpurun_out/s82_${v}_$rep.err
  done
done
