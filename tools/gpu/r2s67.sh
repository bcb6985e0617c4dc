#!/bin/bash
# packet ray cast: certified f32 hit pre-test (b200) vs exact-only (nopf)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -k "ray or packet or c2 or c5 or handoff or acceptance" > gpurun_out/s67_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s67_pytest.log
for v in b200 nopf b200 nopf; do
  echo "== $v" >> gpurun_out/s67_probe.txt
  FHV_LIB=paper_2211_15460_b200/libfhv_$v.so timeout 600 python tools/ray_probe.py >> gpurun_out/s67_probe.txt 2>&1
  FHV_LIB=paper_2211_15460_b200/libfhv_$v.so timeout 600 python tools/ray_probe.py --c5 --reps 2 2>&1 | head -1 >> gpurun_out/s67_probe.txt
done
