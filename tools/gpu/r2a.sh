set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02a_fast.json 2> gpurun_out/r02a_fast.err
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --exact-order > gpurun_out/r02a_exact.json 2> gpurun_out/r02a_exact.err
tail -c 3000 gpurun_out/r02a_fast.json gpurun_out/r02a_exact.json
