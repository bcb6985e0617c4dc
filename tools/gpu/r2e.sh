python -m pytest -x -q tests/test_gpu_parity.py -k "exact_order or big_leaves or huge or levels_one or fast" 2>&1 | tail -3
ncu --set full --import-source on --clock-control none -k regex:k_leaf_fix -c 1 -o gpurun_out/r02e_fix python bench.py --steps 2 --warmup 1 --profile-only --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out
