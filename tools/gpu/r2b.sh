set -x
python -m pytest -x -q tests/test_gpu_parity.py -k "exact_order or big_leaves or huge or levels_one or fast" 2>&1 | tail -15
python -m pytest -x -q -s tests/test_gpu_fullsize.py -k c3 2>&1 | tail -8
python -m pytest -x -q tests/test_gpu_spec.py tests/test_gpu_api.py tests/test_scene_pinning.py 2>&1 | tail -8
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02b.json 2> gpurun_out/r02b.err
tail -c 1500 gpurun_out/r02b.err
