#!/bin/bash
mkdir -p gpurun_out
for v in b200 pipe0 b200 pipe0; do
  echo "== $v" >> gpurun_out/s24_probe.txt
  FHV_LIB=paper_2211_15460_b200/libfhv_$v.so timeout 600 python tools/ray_probe.py >> gpurun_out/s24_probe.txt 2>&1
  FHV_LIB=paper_2211_15460_b200/libfhv_$v.so timeout 600 python tools/ray_probe.py --c5 --reps 2 2>&1 | head -1 >> gpurun_out/s24_probe.txt
done
timeout 900 python -m pytest tests -m gpu -x -q -k "ray or packet or big_leaves or fullsize" > gpurun_out/s24_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s24_pytest.log
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/s24_c3.jsonl 2> gpurun_out/s24_c3.err
