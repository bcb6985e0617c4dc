#!/bin/bash
mkdir -p gpurun_out
for v in b200 prev b200 prev; do
  echo "== $v" >> gpurun_out/s41_probe.txt
  FHV_LIB=paper_2211_15460_b200/libfhv_$v.so timeout 600 python tools/ray_probe.py >> gpurun_out/s41_probe.txt 2>&1
  FHV_LIB=paper_2211_15460_b200/libfhv_$v.so timeout 600 python tools/ray_probe.py --c5 --reps 2 2>&1 | head -1 >> gpurun_out/s41_probe.txt
done
timeout 900 python -m pytest tests -m gpu -x -q -k "ray or packet or fullsize or acceptance" > gpurun_out/s41_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s41_pytest.log
