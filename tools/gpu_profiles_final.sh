#!/bin/bash
# ncu --set full of every kernel family on the current code (round-end evidence)
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:grid_rk4 -c 1 -o gpurun_out/fin_stream_n1e4 -f python bench.py --steps 1 --warmup 0 --rk4-steps 10 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:reg_rk4 -c 1 -o gpurun_out/fin_reg_n1000 -f python bench.py --workload n1000 --steps 1 --warmup 0 --rk4-steps 300 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:ens_rk4 -c 1 -o gpurun_out/fin_ens512 -f python bench.py --workload ens512 --steps 1 --warmup 0 --rk4-steps 20 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:tiny_rk4 -c 1 -o gpurun_out/fin_tiny_n1 -f python bench.py --workload n1 --steps 1 --warmup 0 --rk4-steps 20000 --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin_launches_default.csv python bench.py --steps 2 --warmup 1 --rk4-steps 50 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out/fin_*
