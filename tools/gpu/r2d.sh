python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02d.json 2> gpurun_out/r02d.err
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:leaf -c 20 --csv --log-file gpurun_out/r02d_leaf.csv python bench.py --steps 2 --warmup 1 --profile-only --no-cpu-baseline > /dev/null 2>&1
tail -c 600 gpurun_out/r02d.err
