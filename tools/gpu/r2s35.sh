#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_emit_fast|k_leaf_fix|k_raster" -c 3 --launch-skip 0 -o gpurun_out/s35_c4 -f python bench.py --config C4 --steps 1 --warmup 1 --no-cpu-baseline --no-graph > gpurun_out/s35_ncu.log 2>&1
