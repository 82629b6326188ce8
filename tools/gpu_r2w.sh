#!/bin/bash
# call w: MULTI phases with system- vs gpu-scope exchange fences (logical ranks); n1 sanitizer case
mkdir -p gpurun_out/w
O=gpurun_out/w
for lib in libsto_b200_timeline.so libsto_b200_timeline_gpuscope.so; do for w in 1 2 8; do echo "$lib world=$w"; STO_TL_LIB=$lib STO_L2_KEEP_MB=0 timeout 300 python tools/multi_timeline.py 10000 $w 2>&1 | tail -1; done; done > $O/timeline_scope.txt; cat $O/timeline_scope.txt
CASES="tiny_n1_spec" SAN_TIMEOUT=300 timeout 900 bash tools/sanitize.sh memcheck synccheck racecheck > /dev/null 2>&1; cp -r gpurun_out/sanitize $O/; cut -c1-160 $O/sanitize/summary.txt
