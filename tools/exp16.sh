mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_shard.py -q -x -m gpu -k "ray or c2 or c5" > gpurun_out/exp16_pytest.log 2>&1
for r in 1 2; do
timeout 600 python bench.py --config C2 --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/exp16_C2_$r.jsonl 2>&1
done
timeout 600 python bench.py --config C5 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/exp16_C5.jsonl 2>&1
