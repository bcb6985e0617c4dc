python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02m.json 2> gpurun_out/r02m.err
FHV_EXACT_MATH=1 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02m_exact.json 2>&1
python bench.py --config C4 --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/r02m_c4.json 2>&1
FHV_EXACT_MATH=1 python bench.py --config C4 --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/r02m_c4_exact.json 2>&1
