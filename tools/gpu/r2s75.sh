#!/bin/bash
# rank scan in the directory launch from the counting pass's item tile totals vs look-back (prev)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -k "spec or pofa or fullsize or parity or shard" > gpurun_out/s75_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s75_pytest.log
for rep in 1 2; do
  for v in b200 prev; do
    FHV_LIB=paper_2211_15460_b200/libfhv_$v.so timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/s75_${v}_$rep.jsonl 2> gpurun_out/s75_${v}_$rep.err
  done
done
