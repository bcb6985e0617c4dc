#!/bin/bash
# directory offsets: plain register stores (b200) vs TMA tensor store (tmas)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -k "pofa or fullsize or parity or spec or shard or dir" > gpurun_out/s72_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s72_pytest.log
for rep in 1 2; do
  for v in b200 tmas; do
    FHV_LIB=paper_2211_15460_b200/libfhv_$v.so timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/s72_${v}_$rep.jsonl 2> gpurun_out/s72_${v}_$rep.err
  done
done
