mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "splat" > gpurun_out/exp7_pytest.log 2>&1
timeout 300 python bench.py --steps 30 --no-cpu-baseline > gpurun_out/exp7_bench.jsonl 2> gpurun_out/exp7_bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_dir_tiles|k_splat|k_job_setup" --launch-skip 15 -c 5 -o gpurun_out/exp7_full -f python bench.py --steps 1 --warmup 3 --profile-only > gpurun_out/exp7_ncu.log 2>&1
