#!/bin/bash
# call y: MULTI scratch staging (sharded tests, timeline, cost); long fuzz campaign with statistics
mkdir -p gpurun_out/y
O=gpurun_out/y
timeout 1200 python -m pytest tests/test_gpu_sharded.py -m gpu -q -x -rf > $O/tests_sharded.log 2>&1; tail -2 $O/tests_sharded.log
for w in 1 2 8; do STO_L2_KEEP_MB=0 timeout 300 python tools/multi_timeline.py 10000 $w 2>&1 | tail -1; done > $O/timeline.txt; cat $O/timeline.txt
STO_L2_KEEP_MB=0 timeout 600 python tools/exchange_cost.py 2000 10000 > $O/xc.jsonl 2> $O/xc.err; cat $O/xc.jsonl
STO_FUZZ_SCALE=40 timeout 3000 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_ensemble.py tests/test_gpu_ensemble_exact.py tests/test_gpu_sharded.py -m gpu -q -rf -k "random" --hypothesis-show-statistics > $O/fuzz.log 2>&1; grep -E "passed|failed|passing|Stopped|runtime" $O/fuzz.log | head -30
