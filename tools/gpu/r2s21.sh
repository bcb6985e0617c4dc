#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s21_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s21_pytest.log
timeout 600 python bench.py --config C2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/s21_c2.jsonl 2> gpurun_out/s21_c2.err
timeout 600 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s21_c4.jsonl 2> gpurun_out/s21_c4.err
