python -m pytest -x -q tests/test_gpu_parity.py -k "exact_order or big_leaves or huge or levels_one or fast" 2>&1 | tail -4
python -m pytest -x -q -s tests/test_gpu_fullsize.py -k c3 2>&1 | grep -i "fix-up\|passed\|failed"
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02c.json 2> gpurun_out/r02c.err
tail -c 1500 gpurun_out/r02c.err
