#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/ray_probe.py > gpurun_out/s2_probe.txt 2>&1
timeout 600 python tools/ray_probe.py --c5 --reps 2 >> gpurun_out/s2_probe.txt 2>&1
