#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "splat or fullsize or parity" > gpurun_out/s48_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s48_pytest.log
timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/s48_new.jsonl 2> gpurun_out/s48_new.err
FHV_SPLAT_REPROJECT=0 timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/s48_old.jsonl 2> gpurun_out/s48_old.err
