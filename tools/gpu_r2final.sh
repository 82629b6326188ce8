#!/bin/bash
# round-2 final closing run: everything (tests, smoke, both arms, every workload, launch list,
# ncu of the default kernel, DRAM traffic of every workload, sanitizers over every family)
bash tools/gpu_r2close.sh final
O=gpurun_out/close_final
rm -f $O/stream_n1e4.ncu-rep.tmp
bash tools/gpu_traffic.sh > /dev/null 2>&1; cp gpurun_out/traffic_*.csv $O/ 2>/dev/null
SAN_TIMEOUT=240 timeout 3600 bash tools/sanitize.sh memcheck synccheck racecheck > /dev/null 2>&1; cp -r gpurun_out/sanitize $O/; cut -c1-120 $O/sanitize/summary.txt | awk '{print $1, $2, $3, $4}' | sort | uniq -c | sort -rn | head -5
python tools/ncu_summary.py $O/stream_n1e4.ncu-rep > $O/ncu_stream_n1e4.txt 2>&1; rm -f $O/stream_n1e4.ncu-rep
