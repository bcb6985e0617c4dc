#!/bin/bash
# ncu --set full of the C3 step's raster / emit / fix / splat kernels (line-level)
NCU_FILTER='-k regex:k_(raster|emit|leaf_fix|splat|job_setup) --launch-skip 8 -c 8' STAGES="full" bash tools/gpu_round.sh s13
