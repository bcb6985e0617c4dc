mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_stage_scatter|k_raster" --launch-skip 6 -c 2 -o gpurun_out/exp20_stage -f python bench.py --steps 1 --warmup 4 --profile-only > gpurun_out/exp20_ncu.log 2>&1
