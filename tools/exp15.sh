mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -m gpu -k "ray or c2 or c5 or huge" > gpurun_out/exp15_pytest.log 2>&1
for r in 1 2; do
timeout 600 python bench.py --config C2 --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/exp15_C2_$r.jsonl 2>&1
done
