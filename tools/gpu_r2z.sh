#!/bin/bash
mkdir -p gpurun_out/z
O=gpurun_out/z
for w in 1 2 8; do echo "X0 world=$w"; STO_LIB=x STO_TL_LIB=libsto_b200_timeline_X0.so STO_L2_KEEP_MB=0 timeout 300 python tools/multi_timeline.py 10000 $w 2>&1 | tail -1; done > $O/timeline_x0.txt; cat $O/timeline_x0.txt
