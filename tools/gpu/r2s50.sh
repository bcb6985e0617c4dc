#!/bin/bash
# A/B: leaf-fix counting unroll / next-tile rank prefetch; raster grid CTAs per SM 16 / 32 / 64
mkdir -p gpurun_out
for rep in 1 2; do
  for v in nopf fixu fixp b200 ps32 ps64; do
    FHV_LIB=paper_2211_15460_b200/libfhv_$v.so timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/s50_${v}_$rep.jsonl 2> gpurun_out/s50_${v}_$rep.err
  done
done
for v in b200 ps64; do
  FHV_LIB=paper_2211_15460_b200/libfhv_$v.so timeout 600 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s50_c4_$v.jsonl 2> gpurun_out/s50_c4_$v.err
done
timeout 900 python -m pytest tests -m gpu -x -q -k "pofa or fullsize or order or fix" > gpurun_out/s50_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s50_pytest.log
