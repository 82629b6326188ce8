#!/bin/bash
# call aa: physical-layout exchange + one system fence per role: sharded tests, timeline, cost
mkdir -p gpurun_out/aa
O=gpurun_out/aa
timeout 1200 python -m pytest tests/test_gpu_sharded.py -m gpu -q -x -rf > $O/tests_sharded.log 2>&1; tail -2 $O/tests_sharded.log
for w in 1 2 8; do STO_L2_KEEP_MB=0 timeout 300 python tools/multi_timeline.py 10000 $w 2>&1 | tail -1; done > $O/timeline.txt; cat $O/timeline.txt
STO_L2_KEEP_MB=0 timeout 600 python tools/exchange_cost.py 2000 10000 > $O/xc.jsonl 2> $O/xc.err; cat $O/xc.jsonl
