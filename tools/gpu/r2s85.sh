#!/bin/bash
# packet kernel: 3 CTAs/SM budget for the compositing modes
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -k "ray or packet or c2 or c5 or handoff or acceptance or api" > gpurun_out/s85_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s85_pytest.log
for rep in 1 2; do
  timeout 600 python bench.py --config C2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/s85_c2_$rep.jsonl 2> gpurun_out/s85_c2_$rep.err
done
timeout 900 python bench.py --config C5 --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/s85_c5.jsonl 2> gpurun_out/s85_c5.err
