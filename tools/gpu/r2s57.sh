#!/bin/bash
# leaf-counter / cursor clears on a side stream (A/B via FHV_FORK_CLEARS)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s57_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s57_pytest.log
for rep in 1 2; do
  for v in 1 0; do
    FHV_FORK_CLEARS=$v timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/s57_fc${v}_$rep.jsonl 2> gpurun_out/s57_fc${v}_$rep.err
  done
done
for v in 1 0; do
  FHV_FORK_CLEARS=$v timeout 600 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s57_c4_fc$v.jsonl 2> gpurun_out/s57_c4_fc$v.err
done
