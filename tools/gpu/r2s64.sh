#!/bin/bash
# certified plane keys in the counting pass alone (FHV_FAST_COUNT=1) at C3
mkdir -p gpurun_out
FHV_FAST_COUNT=1 timeout 1200 python -m pytest tests -m gpu -x -q -k "pofa or fullsize" > gpurun_out/s64_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s64_pytest.log
for rep in 1 2; do
  for v in 1 0; do
    FHV_FAST_COUNT=$v timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/s64_fc${v}_$rep.jsonl 2> gpurun_out/s64_fc${v}_$rep.err
  done
done
