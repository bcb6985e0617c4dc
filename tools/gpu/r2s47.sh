#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "deep_octrees" > gpurun_out/s47_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s47_pytest.log
