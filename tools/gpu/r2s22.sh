#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_spec.py -x -q > gpurun_out/s22_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s22_pytest.log
