#!/bin/bash
# grid sweeps: fix-up CTAs per SM (8 / 12 / 13 / 26), raster / emission CTAs per SM (8 / 12 / 16)
mkdir -p gpurun_out
for rep in 1 2; do
  for v in b200 f8 f13 f26 r8 r12; do
    FHV_LIB=paper_2211_15460_b200/libfhv_$v.so timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/s70_${v}_$rep.jsonl 2> gpurun_out/s70_${v}_$rep.err
  done
done
