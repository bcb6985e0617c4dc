#!/bin/bash
# fused plan with the job setup's tile totals (no look-back chain) vs the look-back version (prev)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -k "spec or pofa or fullsize or retry or plan" > gpurun_out/s74_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s74_pytest.log
for rep in 1 2; do
  for v in b200 prev; do
    FHV_LIB=paper_2211_15460_b200/libfhv_$v.so timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/s74_${v}_$rep.jsonl 2> gpurun_out/s74_${v}_$rep.err
  done
done
