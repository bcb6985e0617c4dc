#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "handoff or packet or raycast or ray" > gpurun_out/s37_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s37_pytest.log
