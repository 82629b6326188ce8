#!/bin/bash
# ncu --set full of the cluster kernel (N = 100, configs[0]) + launch lists (default bench, n100)
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:clu_rk4 -c 1 -o gpurun_out/e_clu_n100 -f python bench.py --workload n100 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/e_clu.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/e_launches_default.csv python bench.py --steps 2 --warmup 1 --rk4-steps 50 --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/e_launches_n100.csv python bench.py --workload n100 --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out/e_*
