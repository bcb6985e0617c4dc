mkdir -p gpurun_out
for c in C2 C4 C5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 2 > gpurun_out/exp2_$c.jsonl 2> gpurun_out/exp2_$c.err
done
