mkdir -p gpurun_out
for v in b200 nofastdiv; do
  export FHV_LIB=$PWD/paper_2211_15460_b200/libfhv_$v.so
  timeout 300 python bench.py --steps 30 --no-cpu-baseline > gpurun_out/exp5_$v.jsonl 2> gpurun_out/exp5_$v.err
  timeout 300 python bench.py --config C2 --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/exp5_C2_$v.jsonl 2>&1
done
unset FHV_LIB
timeout 300 python tools/host_profile.py 30 > gpurun_out/exp5_hostprof.txt 2>&1
