#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "pofa or fullsize or parity or ppfl or pofl or shard or spec" > gpurun_out/s42_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s42_pytest.log
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/s42_c3.jsonl 2> gpurun_out/s42_c3.err
