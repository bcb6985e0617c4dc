#!/bin/bash
# programmatic dependent launch on the adjacent kernel pairs (FHV_PDL=0: ordinary launches)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s86_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s86_pytest.log
for rep in 1 2; do
  for v in 1 0; do
    FHV_PDL=$v timeout 600 python bench.py --steps 50 --warmup 3 --no-cpu-baseline > gpurun_out/s86_p${v}_$rep.jsonl 2> gpurun_out/s86_p${v}_$rep.err
  done
done
for v in 1 0; do
  FHV_PDL=$v timeout 600 python bench.py --config C5 --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/s86_c5_p$v.jsonl 2> gpurun_out/s86_c5_p$v.err
done
