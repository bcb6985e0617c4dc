#!/bin/bash
# packet ray cast: parity suite + C2 / C5 timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "raycast or ray or acceptance or fullsize or api or shard" > gpurun_out/s1_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s1_pytest.log
timeout 600 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s1_c2.jsonl 2> gpurun_out/s1_c2.err
timeout 900 python bench.py --config C5 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/s1_c5.jsonl 2> gpurun_out/s1_c5.err
