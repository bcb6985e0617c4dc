mkdir -p gpurun_out
for v in b200 ray4 ray6 ray8; do
  export FHV_LIB=$PWD/paper_2211_15460_b200/libfhv_$v.so
  timeout 300 python bench.py --config C2 --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/exp8_C2_$v.jsonl 2>&1
done
