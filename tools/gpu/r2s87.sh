#!/bin/bash
# ray casts into a reused buffer without a clear
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_spec.py -x -q -k "reused_buffer" > gpurun_out/s87_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s87_pytest.log
timeout 600 python bench.py --config C2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/s87_c2.jsonl 2> gpurun_out/s87_c2.err
timeout 900 python bench.py --config C5 --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/s87_c5.jsonl 2> gpurun_out/s87_c5.err
timeout 900 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s87_c4.jsonl 2> gpurun_out/s87_c4.err
