#!/bin/bash
# e2e regression hunt: the r02i build (29fe5ae), the depth-grid build (abd125d), HEAD
mkdir -p gpurun_out
for rep in 1 2; do
  for v in b200 29fe5ae abd125d; do
    FHV_LIB=paper_2211_15460_b200/libfhv_$v.so timeout 600 python bench.py --steps 60 --warmup 3 --no-cpu-baseline > gpurun_out/s76_${v}_$rep.jsonl 2> gpurun_out/s76_${v}_$rep.err
  done
done
