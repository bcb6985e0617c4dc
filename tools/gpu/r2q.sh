ncu --set full --import-source on --clock-control none -k regex:"k_splat_depth_fast|k_splat_index_stored|k_emit|k_raster|k_splat_resolve|k_dir_tiles|k_leaf_fix" -c 8 -o gpurun_out/r02q_full python bench.py --steps 2 --warmup 1 --profile-only --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out/r02q_full.ncu-rep
