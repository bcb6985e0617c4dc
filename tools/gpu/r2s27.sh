#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_shard.py tests/test_gpu_shard_procs.py -x -q > gpurun_out/s27_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s27_pytest.log
