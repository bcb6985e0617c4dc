#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "splat or fullsize or parity" > gpurun_out/s15_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s15_pytest.log
timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/s15_agg.jsonl 2> gpurun_out/s15_agg.err
FHV_SPLAT_AGG=0 timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/s15_base.jsonl 2> gpurun_out/s15_base.err
