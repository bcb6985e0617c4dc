#!/bin/bash
mkdir -p gpurun_out
for nb in 2 3 4; do
  FHV_E2E_BUFFERS=$nb timeout 600 python bench.py --steps 60 --warmup 3 --no-cpu-baseline > gpurun_out/s63_nb$nb.jsonl 2> gpurun_out/s63_nb$nb.err
done
