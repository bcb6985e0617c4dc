mkdir -p gpurun_out
for v in res1 res2 res4; do
  export FHV_LIB=$PWD/paper_2211_15460_b200/libfhv_$v.so
  timeout 300 python bench.py --steps 30 --no-cpu-baseline > gpurun_out/exp12_$v.jsonl 2> gpurun_out/exp12_$v.err
done
unset FHV_LIB
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k splat > gpurun_out/exp12_pytest.log 2>&1
FHV_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/exp12_gloo2.jsonl 2> gpurun_out/exp12_gloo2.err
