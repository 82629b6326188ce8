#!/bin/bash
# ncu evidence for the kernels added/changed in the second half of round 1
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:ens_rk4 -c 1 -o gpurun_out/r01_ens512_v2 -f python bench.py --workload ens512 --steps 1 --warmup 0 --rk4-steps 20 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"pcg64_fill|gemv_kernel" -c 2 -o gpurun_out/r01_build_n1e4 -f python -c "
import sys; sys.path.insert(0,'.')
import paper_2312_01121_b200 as sto; sto.build_topology_device(10000)" > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches_default_b.csv python bench.py --steps 2 --warmup 1 --rk4-steps 50 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep gpurun_out/*.csv
