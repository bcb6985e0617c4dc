#!/bin/bash
mkdir -p gpurun_out
for v in b200 m5 m6; do
  echo "== $v" >> gpurun_out/s8_probe.txt
  FHV_LIB=paper_2211_15460_b200/libfhv_$v.so timeout 600 python tools/ray_probe.py >> gpurun_out/s8_probe.txt 2>&1
  FHV_LIB=paper_2211_15460_b200/libfhv_$v.so timeout 600 python tools/ray_probe.py --c5 --reps 2 2>&1 | head -1 >> gpurun_out/s8_probe.txt
done
