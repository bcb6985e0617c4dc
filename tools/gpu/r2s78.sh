#!/bin/bash
# e2e steps as graph replays (default) vs plain asynchronous calls (FHV_E2E_GRAPH=0)
mkdir -p gpurun_out
for rep in 1 2 3; do
  for v in 1 0; do
    FHV_E2E_GRAPH=$v timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s78_g${v}_$rep.jsonl 2> gpurun_out/s78_g${v}_$rep.err
  done
done
