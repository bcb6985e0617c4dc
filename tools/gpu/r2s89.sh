#!/bin/bash
# splat keys + winners in one allocation, one clear
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -k "splat or fullsize or parity or deferred or gbuffer or api or acceptance" > gpurun_out/s89_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s89_pytest.log
for rep in 1 2; do
  timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/s89_c3_$rep.jsonl 2> gpurun_out/s89_c3_$rep.err
done
