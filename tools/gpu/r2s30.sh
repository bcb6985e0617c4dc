#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_raycast_packet -c 1 -o gpurun_out/s30_c5 -f python tools/ray_probe.py --c5 --reps 1 > gpurun_out/s30_ncu.log 2>&1
