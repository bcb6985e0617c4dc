#!/bin/bash
# splat depth grid fine sweep: 5 / 6 (b200) / 7 / 10 CTAs per SM
mkdir -p gpurun_out
for rep in 1 2; do
  for v in b200 d5 d7 d10; do
    FHV_LIB=paper_2211_15460_b200/libfhv_$v.so timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/s88_${v}_$rep.jsonl 2> gpurun_out/s88_${v}_$rep.err
  done
done
