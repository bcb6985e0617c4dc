#!/bin/bash
# side-stream clears: mode 2 (cursors during the counting pass) vs mode 1 (both during the job setup)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "pofa or spec or fullsize or parity or shard" > gpurun_out/s59_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s59_pytest.log
for rep in 1 2; do
  for v in 2 1; do
    FHV_FORK_CLEARS=$v timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/s59_fc${v}_$rep.jsonl 2> gpurun_out/s59_fc${v}_$rep.err
  done
done
