#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "forced or fullsize or parity" > gpurun_out/s26_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s26_pytest.log
FHV_FAST_MATH=1 timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/s26_fast.jsonl 2> gpurun_out/s26_fast.err
timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/s26_base.jsonl 2> gpurun_out/s26_base.err
timeout 600 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s26_c4.jsonl 2> gpurun_out/s26_c4.err
