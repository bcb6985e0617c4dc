mkdir -p gpurun_out
for r in 1 2; do for v in pf pf2; do
  export FHV_LIB=$PWD/paper_2211_15460_b200/libfhv_$v.so
  timeout 300 python bench.py --steps 30 --no-cpu-baseline > gpurun_out/exp18_${v}_$r.jsonl 2> gpurun_out/exp18_$v.err
done; done
