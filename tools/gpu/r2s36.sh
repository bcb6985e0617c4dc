#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "pofa or fullsize or parity or shard or spec or ppfl or pofl" > gpurun_out/s36_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s36_pytest.log
for c in 0 4 8 16 32; do
  FHV_EMIT_CHUNK=$c timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/s36_c$c.jsonl 2> gpurun_out/s36_c$c.err
done
FHV_EMIT_CHUNK=8 timeout 600 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s36_c4.jsonl 2> gpurun_out/s36_c4.err
