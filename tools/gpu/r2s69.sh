#!/bin/bash
# splat depth pass grid: CTAs per SM 4 / 6 / 8 (b200) / 12 / 16
mkdir -p gpurun_out
for rep in 1 2; do
  for v in b200 d4 d6 d12 d16; do
    FHV_LIB=paper_2211_15460_b200/libfhv_$v.so timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/s69_${v}_$rep.jsonl 2> gpurun_out/s69_${v}_$rep.err
  done
done
for v in b200 d16; do
  FHV_LIB=paper_2211_15460_b200/libfhv_$v.so timeout 600 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s69_c5_$v.jsonl 2> gpurun_out/s69_c5_$v.err
done
