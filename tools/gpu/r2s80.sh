#!/bin/bash
# directory launch stores the fragment total (no D2D copy node)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s80_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s80_pytest.log
for rep in 1 2; do
  timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s80_c3_$rep.jsonl 2> gpurun_out/s80_c3_$rep.err
done
