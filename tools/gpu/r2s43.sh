#!/bin/bash
mkdir -p gpurun_out
for v in b200 prev b200 prev; do
  echo "== $v" >> gpurun_out/s43_probe.txt
  FHV_LIB=paper_2211_15460_b200/libfhv_$v.so timeout 600 python tools/ray_probe.py >> gpurun_out/s43_probe.txt 2>&1
done
timeout 900 python -m pytest tests -m gpu -x -q -k "ray or packet or fullsize or acceptance or pofl or spec" > gpurun_out/s43_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s43_pytest.log
