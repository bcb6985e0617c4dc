#!/bin/bash
# One gpurun call: GPU tests, smoke, bench, reference arm, ncu launch list, ncu --set full of the step.
# usage (from repo root, under gpurun):  STAGES="pytest bench" bash tools/gpu_round.sh TAG [pytest-args]
set -x
TAG=${1:-rX}; shift
STAGES=${STAGES:-"pytest smoke bench ref launches full"}
has() { [[ " $STAGES " == *" $1 "* ]]; }
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
if has pytest; then
  timeout 1500 python -m pytest tests -m gpu -x -q "$@" > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
fi
if has smoke; then
  timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
fi
if has bench; then
  timeout 600 python bench.py ${BENCH_ARGS} > gpurun_out/${TAG}_bench.jsonl 2> gpurun_out/${TAG}_bench.err
fi
if has ref; then
  timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_bench_ref.jsonl 2> gpurun_out/${TAG}_bench_ref.err
fi
if has launches; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv \
      python bench.py --steps 2 --warmup 3 --profile-only > /dev/null 2>&1
fi
if has full; then
  timeout 900 ncu --set full --clock-control none --import-source on ${NCU_FILTER:---launch-skip 44 -c 11} -o gpurun_out/${TAG}_full -f \
      python bench.py --steps 1 --warmup 3 --profile-only > gpurun_out/${TAG}_ncu_full.log 2>&1
fi
# keep gpurun_out under the 64 MiB copy-back limit
find gpurun_out -name '*.ncu-rep' -size +45M -delete
