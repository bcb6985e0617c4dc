#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_indexed.py tests/test_gpu_parity.py::test_forced_arithmetic_paths_bit_exact tests/test_gpu_api.py -x -q > gpurun_out/r02b_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02b_pytest.log
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/r02b_bench.jsonl 2> gpurun_out/r02b_bench.err
timeout 600 python bench.py --steps 50 --warmup 5 --upload soup --no-cpu-baseline > gpurun_out/r02b_bench_soup.jsonl 2> gpurun_out/r02b_bench_soup.err
