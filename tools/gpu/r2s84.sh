#!/bin/bash
# packet ray cast register budget: 4 CTAs (128 regs, default) vs 3 (170) vs 2 (255)
mkdir -p gpurun_out
for v in b200 pm3 pm2 b200 pm3 pm2; do
  echo "== $v" >> gpurun_out/s84_probe.txt
  FHV_LIB=paper_2211_15460_b200/libfhv_$v.so timeout 600 python tools/ray_probe.py >> gpurun_out/s84_probe.txt 2>&1
  FHV_LIB=paper_2211_15460_b200/libfhv_$v.so timeout 600 python tools/ray_probe.py --c5 --reps 2 2>&1 | head -1 >> gpurun_out/s84_probe.txt
done
