#!/bin/bash
# striped fused job scan + item expansion (8 / 4 jobs per thread) vs separate (FHV_FUSED_EXPAND=0)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "spec or pofa or fullsize or retry or plan" > gpurun_out/s55_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s55_pytest.log
for rep in 1 2; do
  FHV_FUSED_EXPAND=0 timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/s55_sep_$rep.jsonl 2> gpurun_out/s55_sep_$rep.err
  for v in b200 e4; do
    FHV_LIB=paper_2211_15460_b200/libfhv_$v.so timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/s55_${v}_$rep.jsonl 2> gpurun_out/s55_${v}_$rep.err
  done
done
