python bench.py --config C4 --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/r02k_c4.json 2> gpurun_out/r02k_c4.err
FHV_EXACT_MATH=1 python bench.py --config C4 --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/r02k_c4_exact.json 2>&1
tail -3 gpurun_out/r02k_c4.err
