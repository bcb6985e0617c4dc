mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -m gpu -k "ray or c2 or c5" > gpurun_out/exp3_pytest.log 2>&1
timeout 600 python bench.py --config C2 --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/exp3_C2.jsonl 2> gpurun_out/exp3_C2.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_raycast -c 1 -o gpurun_out/exp3_ray -f python bench.py --config C2 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/exp3_ncu.log 2>&1
