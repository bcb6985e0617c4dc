#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "c4_depth_complexity_raycast" > gpurun_out/s46_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s46_pytest.log
