#!/bin/bash
# call s: MULTI staging unrolled (cost + timeline + sharded tests); exact ensemble BV 1/2/4 tiles
mkdir -p gpurun_out/s
O=gpurun_out/s
STO_L2_KEEP_MB=0 timeout 600 python tools/exchange_cost.py 2000 10000 > $O/xc.jsonl 2> $O/xc.err; cat $O/xc.jsonl; tail -2 $O/xc.err
for w in 1 2 8; do STO_L2_KEEP_MB=0 timeout 300 python tools/multi_timeline.py 10000 $w 2>&1 | tail -1; done > $O/timeline.txt; cat $O/timeline.txt
for bv in 1 2 4; do STO_EX_BV=$bv timeout 900 python bench.py --workload ens512_exact --steps 3 --warmup 2 --no-cpu-baseline > $O/bench_exact_bv$bv.json 2> $O/bench_exact_bv$bv.err; python -c "
import json; d=json.loads(open('$O/bench_exact_bv$bv.json').read()); print('BV=$bv', '%.4g'%d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'])"; tail -1 $O/bench_exact_bv$bv.err; done
timeout 1200 python -m pytest tests/test_gpu_sharded.py -m gpu -q -x -rf > $O/tests_sharded.log 2>&1; tail -2 $O/tests_sharded.log
for bv in 1 4; do STO_EX_BV=$bv timeout 1200 python -m pytest tests/test_gpu_ensemble_exact.py -m gpu -q -x -rf > $O/tests_exact_bv$bv.log 2>&1; tail -2 $O/tests_exact_bv$bv.log; done
