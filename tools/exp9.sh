mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_dir|k_tile_prefix" --launch-skip 9 -c 3 -o gpurun_out/exp9_dir -f python bench.py --steps 1 --warmup 3 --profile-only > gpurun_out/exp9_ncu.log 2>&1
