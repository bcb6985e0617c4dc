python -m pytest -x -q tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_spec.py tests/test_gpu_acceptance.py 2>&1 | tail -2
FHV_FAST_MATH=1 python -m pytest -x -q tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_spec.py 2>&1 | tail -2
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02n.json 2> gpurun_out/r02n.err
python bench.py --config C4 --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/r02n_c4.json 2>&1
