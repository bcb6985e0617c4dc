#!/bin/bash
# speculative plan: fused job scan + item expansion (A/B via FHV_FUSED_EXPAND)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s54_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s54_pytest.log
for rep in 1 2; do
  for v in 1 0; do
    FHV_FUSED_EXPAND=$v timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/s54_fe${v}_$rep.jsonl 2> gpurun_out/s54_fe${v}_$rep.err
  done
done
for v in 1 0; do
  FHV_FUSED_EXPAND=$v timeout 600 python bench.py --config C2 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/s54_c2_fe$v.jsonl 2> gpurun_out/s54_c2_fe$v.err
done
