mkdir -p gpurun_out
for r in 1 2; do
timeout 600 python bench.py --config C2 --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/exp13_C2_$r.jsonl 2>&1
done
timeout 600 python bench.py --config C2 --steps 5 --warmup 2 > gpurun_out/exp13_C2_cpu.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -m gpu -k "ray or c2 or c5" > gpurun_out/exp13_pytest.log 2>&1
