#!/bin/bash
# packet ray-cast knob sweep: per-lane hit slots, deferred-record queue
mkdir -p gpurun_out
for v in b200 hits_2 hits_8 buf_8 buf_16; do
  echo "== $v" >> gpurun_out/s23_probe.txt
  FHV_LIB=paper_2211_15460_b200/libfhv_$v.so timeout 600 python tools/ray_probe.py >> gpurun_out/s23_probe.txt 2>&1
  FHV_LIB=paper_2211_15460_b200/libfhv_$v.so timeout 600 python tools/ray_probe.py --c5 --reps 2 2>&1 | head -1 >> gpurun_out/s23_probe.txt
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "packet or big_leaves" > gpurun_out/s23_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s23_pytest.log
