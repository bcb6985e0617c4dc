python -m pytest -x -q tests/test_gpu_parity.py tests/test_gpu_fullsize.py -k "c3 or exact or levels or stores" 2>&1 | tail -1
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02s.json 2> gpurun_out/r02s.err
FHV_DIR_STREAM=0 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02s_old.json 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_dir" -c 1 -o gpurun_out/r02s_dir python bench.py --steps 2 --warmup 1 --profile-only --no-cpu-baseline > /dev/null 2>&1
