#!/bin/bash
mkdir -p gpurun_out
FHV_FAST_MATH=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_emit_fast -c 1 --launch-skip 2 -o gpurun_out/s25_fast -f python bench.py --steps 1 --warmup 3 --profile-only > gpurun_out/s25_ncu.log 2>&1
