#!/bin/bash
# splat depth pass: load-test before each RED.MIN (lt) vs plain reductions
mkdir -p gpurun_out
FHV_LIB=paper_2211_15460_b200/libfhv_lt.so timeout 1200 python -m pytest tests -m gpu -x -q -k "splat or fullsize" > gpurun_out/s60_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s60_pytest.log
for rep in 1 2; do
  for v in b200 lt; do
    FHV_LIB=paper_2211_15460_b200/libfhv_$v.so timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/s60_${v}_$rep.jsonl 2> gpurun_out/s60_${v}_$rep.err
  done
done
for v in b200 lt; do
  FHV_LIB=paper_2211_15460_b200/libfhv_$v.so timeout 600 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s60_c5_$v.jsonl 2> gpurun_out/s60_c5_$v.err
done
