#!/bin/bash
# C3 bench line x3 (the e2e leg varies run to run) + the PCIe probe x3
mkdir -p gpurun_out
for rep in 1 2 3; do
  timeout 600 python bench.py > gpurun_out/s77_c3_$rep.jsonl 2> gpurun_out/s77_c3_$rep.err
  timeout 300 python tools/pcie_probe.py > gpurun_out/s77_pcie_$rep.txt 2>&1
done
