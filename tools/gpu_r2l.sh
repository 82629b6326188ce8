#!/bin/bash
# round 2 session 3, call l: speculative division (tiny kernel), ensemble record-step stop,
# logical-order vectorised sharded exchange; exchange cost; ensemble horizon bar; n1 bench
mkdir -p gpurun_out/l
O=gpurun_out/l
timeout 1500 python -m pytest tests/test_gpu_division.py tests/test_gpu_ensemble.py tests/test_gpu_sharded.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -q -rf --durations=10 > $O/tests.log 2>&1; tail -4 $O/tests.log
timeout 600 python bench.py --workload n1 > $O/bench_n1.json 2> $O/bench_n1.err; head -c 400 $O/bench_n1.json; echo
timeout 600 python tools/exchange_cost.py 2000 10000 > $O/exchange_cost.jsonl 2> $O/exchange_cost.err; cat $O/exchange_cost.jsonl
timeout 1200 python tools/ens_horizon_bar.py 0,511 > $O/ens_bar.json 2> $O/ens_bar.err; cat $O/ens_bar.json
