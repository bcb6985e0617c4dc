#!/bin/bash
# A/B: leaf-fix load hoisting (nopf vs prev), next-group lookahead (b200 vs nopf), persistent raster grid (pfp)
mkdir -p gpurun_out
for rep in 1 2; do
  for v in prev nopf b200 pfp; do
    FHV_LIB=paper_2211_15460_b200/libfhv_$v.so timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/s49_${v}_$rep.jsonl 2> gpurun_out/s49_${v}_$rep.err
  done
done
for v in prev b200 pfp; do
  FHV_LIB=paper_2211_15460_b200/libfhv_$v.so timeout 600 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s49_c4_$v.jsonl 2> gpurun_out/s49_c4_$v.err
done
timeout 900 python -m pytest tests -m gpu -x -q -k "pofa or fullsize or parity or spec" > gpurun_out/s49_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s49_pytest.log
