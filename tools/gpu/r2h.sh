python -m pytest -x -q tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_acceptance.py tests/test_gpu_spec.py 2>&1 | tail -4
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02h.json 2> gpurun_out/r02h.err
FHV_EXACT_MATH=1 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02h_exactmath.json 2>&1
tail -c 800 gpurun_out/r02h.err
