python -m pytest -x -q tests/test_gpu_parity.py tests/test_gpu_fullsize.py -k "c3 or exact or fast or huge or levels" 2>&1 | tail -2
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02j.json 2> gpurun_out/r02j.err
FHV_LIB=$PWD/paper_2211_15460_b200/libfhv_minb2.so python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02j_minb2.json 2>&1
