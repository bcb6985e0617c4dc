python -m pytest -x -q tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_shard.py -k "c3 or exact or levels or stores or shard" 2>&1 | tail -1
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02t.json 2> gpurun_out/r02t.err
FHV_LIB=$PWD/paper_2211_15460_b200/libfhv_dir4.so python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02t_4.json 2>&1
FHV_LIB=$PWD/paper_2211_15460_b200/libfhv_dir1.so python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02t_1.json 2>&1
FHV_LIB=$PWD/paper_2211_15460_b200/libfhv_dir4.so python -m pytest -x -q tests/test_gpu_parity.py -k "exact or levels or stores" 2>&1 | tail -1
