#!/bin/bash
# knob sweep: splat resolve unroll / min blocks, fix-up warps per CTA
mkdir -p gpurun_out
for rep in 1 2; do
  for v in b200 ru1 ru4 rm3 rm1 fw8 fw2; do
    FHV_LIB=paper_2211_15460_b200/libfhv_$v.so timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/s52_${v}_$rep.jsonl 2> gpurun_out/s52_${v}_$rep.err
  done
done
