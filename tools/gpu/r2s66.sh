#!/bin/bash
# certified POFA emission: column-major walk of whole-item groups (C4) vs flat
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -k "c4_depth_complex_ppfl or forced or big_leaves or pofa" > gpurun_out/s66_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s66_pytest.log
for rep in 1 2; do
  for v in b200 nocm; do
    FHV_LIB=paper_2211_15460_b200/libfhv_$v.so timeout 600 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s66_c4_${v}_$rep.jsonl 2> gpurun_out/s66_c4_${v}_$rep.err
  done
done
timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/s66_c3.jsonl 2> gpurun_out/s66_c3.err
