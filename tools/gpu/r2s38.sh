#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "random_cameras" > gpurun_out/s38_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s38_pytest.log
