#!/bin/bash
# item-rank scan fused into the directory launch; fix-up 2 warps per CTA
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s53_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s53_pytest.log
for rep in 1 2; do
  for v in prev b200; do
    FHV_LIB=paper_2211_15460_b200/libfhv_$v.so timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/s53_${v}_$rep.jsonl 2> gpurun_out/s53_${v}_$rep.err
  done
done
