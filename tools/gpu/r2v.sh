python -m pytest -x -q tests/test_gpu_shard.py tests/test_gpu_shard_procs.py 2>&1 | tail -15
