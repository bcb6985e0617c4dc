python -m pytest -x -q tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_acceptance.py tests/test_gpu_next.py tests/test_gpu_spec.py 2>&1 | tail -2
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02r.json 2> gpurun_out/r02r.err
tail -c 400 gpurun_out/r02r.err
