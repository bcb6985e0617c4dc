#!/bin/bash
# L2-only (ld.global.cg) directory and job-record loads in the raster passes vs through L1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "pofa or fullsize or parity" > gpurun_out/s61_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s61_pytest.log
for rep in 1 2; do
  for v in b200 jl1 l1; do
    FHV_LIB=paper_2211_15460_b200/libfhv_$v.so timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/s61_${v}_$rep.jsonl 2> gpurun_out/s61_${v}_$rep.err
  done
done
for v in b200 l1; do
  FHV_LIB=paper_2211_15460_b200/libfhv_$v.so timeout 600 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s61_c4_$v.jsonl 2> gpurun_out/s61_c4_$v.err
done
