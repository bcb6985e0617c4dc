#!/bin/bash
# A/B: one-sweep 128-bit CAS splat vs the two-pass exact splat
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "splat or fullsize or parity or gbuffer or shard" > gpurun_out/s51_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s51_pytest.log
for rep in 1 2; do
  for v in 1 0; do
    FHV_SPLAT_CAS=$v timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/s51_cas${v}_$rep.jsonl 2> gpurun_out/s51_cas${v}_$rep.err
  done
done
for v in 1 0; do
  FHV_SPLAT_CAS=$v timeout 600 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s51_c5_cas$v.jsonl 2> gpurun_out/s51_c5_cas$v.err
done
