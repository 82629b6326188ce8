#!/bin/bash
# call r: ncu of the MULTI kernel (logical world 2, N=1e4); cluster sweep at N=100
mkdir -p gpurun_out/r
O=gpurun_out/r
STO_L2_KEEP_MB=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:grid_rk4 -c 1 -o $O/multi_w2 -f python tools/multi_run.py 10000 2 20 > $O/ncu_multi.log 2>&1; tail -1 $O/ncu_multi.log
timeout 1200 python tools/clu_sweep.py 100 > $O/clu_sweep_100.log 2>&1; cat $O/clu_sweep_100.log
