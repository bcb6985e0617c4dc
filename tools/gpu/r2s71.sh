#!/bin/bash
# raster / emission occupancy: 4 CTAs of 256 (64 registers) and 128-thread CTAs
mkdir -p gpurun_out
for rep in 1 2; do
  for v in b200 m4 m4b b128; do
    FHV_LIB=paper_2211_15460_b200/libfhv_$v.so timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/s71_${v}_$rep.jsonl 2> gpurun_out/s71_${v}_$rep.err
  done
done
