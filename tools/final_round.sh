#!/bin/bash
# Full measurement pass of the current build (one gpurun call):
#   pytest -m gpu, smoke, C3 bench (driver default), reference arm, the other
#   BASELINE configs, ncu launch list and ncu --set full of one C3 step.
TAG=${1:-rX}
mkdir -p gpurun_out
# every timed run before the first ncu session (a box that has run ncu showed
# host-side slowdowns in later benches)
STAGES="pytest smoke bench ref" bash tools/gpu_round.sh $TAG
timeout 900 python bench.py --config C2 --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_C2.jsonl 2> gpurun_out/${TAG}_bench_C2.err
timeout 900 python bench.py --config C4 --steps 10 --warmup 3 > gpurun_out/${TAG}_bench_C4.jsonl 2> gpurun_out/${TAG}_bench_C4.err
timeout 900 python bench.py --config C5 --steps 3 --warmup 1 > gpurun_out/${TAG}_bench_C5.jsonl 2> gpurun_out/${TAG}_bench_C5.err
STAGES="launches" bash tools/gpu_round.sh $TAG
# one C3 step's 10 kernels (job setup, plan, count, directory + ranks,
# emission, fix-up x2, splat x3) after the warm-up steps (the first one
# first two synchronous: 9 matching launches each, then an asynchronous one)
NCU_FILTER='-k regex:k_(job_setup|item_scan|raster|dir_tma|emit|leaf_fix|splat) --launch-skip 28 -c 10' \
    STAGES="full" bash tools/gpu_round.sh $TAG
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_raycast -c 1 -o gpurun_out/${TAG}_ray -f \
    python bench.py --config C2 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/${TAG}_ray_ncu.log 2>&1
timeout 300 python tools/host_profile.py 30 > gpurun_out/${TAG}_hostprof.txt 2>&1
find gpurun_out -name '*.ncu-rep' -size +45M -delete
