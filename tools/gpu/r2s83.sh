#!/bin/bash
# fewer memset nodes in the asynchronous build (counters fresh from its control-block reset)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s83_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s83_pytest.log
for rep in 1 2; do
  for v in b200 prev; do
    FHV_LIB=paper_2211_15460_b200/libfhv_$v.so timeout 600 python bench.py --steps 50 --warmup 3 --no-cpu-baseline > gpurun_out/s83_${v}_$rep.jsonl 2> gpurun_out/s83_${v}_$rep.err
  done
done
