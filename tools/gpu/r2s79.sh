#!/bin/bash
# tickets stored by the ticket kernel through the pinned mapping (default) vs a stream-ordered copy
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s79_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s79_pytest.log
for rep in 1 2 3; do
  for v in 1 0; do
    FHV_TICKET_DIRECT=$v timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s79_t${v}_$rep.jsonl 2> gpurun_out/s79_t${v}_$rep.err
  done
done
for v in 1 0; do
  FHV_TICKET_DIRECT=$v timeout 600 python bench.py --config C2 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/s79_c2_t$v.jsonl 2> gpurun_out/s79_c2_t$v.err
done
