#!/bin/bash
# ensemble: bench + timeline + one ncu --set full capture of ens_rk4_kernel
bash tools/gpu_ens.sh
ncu --set full --clock-control none --import-source on -k regex:ens_rk4 -c 1 -o gpurun_out/ens512 -f python bench.py --workload ens512 --steps 1 --warmup 0 --rk4-steps 20 --no-cpu-baseline > gpurun_out/ncu_ens.log 2>&1; tail -2 gpurun_out/ncu_ens.log
