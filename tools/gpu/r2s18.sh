#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/ray_probe.py > gpurun_out/s18_probe.txt 2>&1
timeout 600 python tools/ray_probe.py --c5 --reps 2 >> gpurun_out/s18_probe.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "raycast or ray or acceptance or fullsize or api or shard" > gpurun_out/s18_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s18_pytest.log
