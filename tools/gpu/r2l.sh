ncu --set full --import-source on --clock-control none -k regex:"k_emit" -c 1 -o gpurun_out/r02l_c4fast python bench.py --config C4 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
FHV_EXACT_MATH=1 ncu --set full --import-source on --clock-control none -k regex:"k_emit" -c 1 -o gpurun_out/r02l_c4exact python bench.py --config C4 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out
