#!/bin/bash
# session re-entry check: GPU suite, C3 and C2 bench on the rebuilt tree
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s0_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s0_pytest.log
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/s0_c3.jsonl 2> gpurun_out/s0_c3.err
timeout 600 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s0_c2.jsonl 2> gpurun_out/s0_c2.err
