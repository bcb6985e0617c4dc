python -m pytest -x -q tests/test_gpu_parity.py -k "exact_order or big_leaves or huge or levels" 2>&1 | tail -1
python -m pytest -x -q -s tests/test_gpu_fullsize.py -k c3 2>&1 | grep -i "fix-up\|passed\|failed"
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02o.json 2> gpurun_out/r02o.err
python bench.py --config C4 --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/r02o_c4.json 2>&1
