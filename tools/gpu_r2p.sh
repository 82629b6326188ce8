#!/bin/bash
# call p: sharded exchange A/B (pre-change X0 vs current) and per-phase timeline
mkdir -p gpurun_out/p
O=gpurun_out/p
for v in X0 C; do lib=libsto_b200_$v.so; [ $v = C ] && lib=libsto_b200.so
  STO_LIB=$lib STO_L2_KEEP_MB=0 timeout 600 python tools/exchange_cost.py 10000 > $O/xc_$v.jsonl 2> $O/xc_$v.err; echo "== $v"; cat $O/xc_$v.jsonl; tail -2 $O/xc_$v.err; done
for w in 1 2 8; do STO_L2_KEEP_MB=0 timeout 300 python tools/multi_timeline.py 10000 $w 2>&1 | tail -2; done > $O/timeline.txt; cat $O/timeline.txt
