#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "forced or fullsize or big_leaves or huge or c4" > gpurun_out/s39_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s39_pytest.log
for v in b200 pipe0; do
  FHV_LIB=paper_2211_15460_b200/libfhv_$v.so timeout 600 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s39_c4_$v.jsonl 2> gpurun_out/s39_c4_$v.err
done
