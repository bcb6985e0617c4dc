#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_raycast_packet -c 1 -o gpurun_out/s40_pkt -f python tools/ray_probe.py --reps 1 > gpurun_out/s40_ncu.log 2>&1
