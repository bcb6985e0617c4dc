set -x
mkdir -p gpurun_out
for v in default minb4; do
  if [ $v = default ]; then unset FHV_LIB; else export FHV_LIB=$PWD/paper_2211_15460_b200/libfhv_$v.so; fi
  timeout 300 python bench.py --steps 30 --no-cpu-baseline > gpurun_out/exp1_$v.jsonl 2> gpurun_out/exp1_$v.err
done
unset FHV_LIB
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/exp1_parity.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_emit|k_raster|k_splat_depth|k_dir_tiles" --launch-skip 12 -c 4 -o gpurun_out/exp1_full -f python bench.py --steps 1 --warmup 3 --profile-only > gpurun_out/exp1_ncu.log 2>&1
find gpurun_out -name '*.ncu-rep' -size +45M -delete
