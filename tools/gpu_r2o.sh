#!/bin/bash
# call o: exact ensemble with 8U x 64 tiles (U = 7 at configs[3]); exchange cost without the L2 slice
mkdir -p gpurun_out/o
O=gpurun_out/o
timeout 1500 python -m pytest tests/test_gpu_ensemble_exact.py -m gpu -q -x -rf --durations=5 > $O/tests.log 2>&1; tail -12 $O/tests.log
for u in 7 4; do STO_EX_U=$u timeout 900 python bench.py --workload ens512_exact --steps 3 --warmup 2 --no-cpu-baseline > $O/bench_exact_u$u.json 2> $O/bench_exact_u$u.err; python -c "
import json; d=json.loads(open('$O/bench_exact_u$u.json').read()); print('U=$u', '%.4g'%d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'])"; done
STO_L2_KEEP_MB=0 timeout 600 python tools/exchange_cost.py 2000 10000 > $O/exchange_cost_nol2.jsonl 2> $O/exchange_cost.err; cat $O/exchange_cost_nol2.jsonl
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ens_exact -c 1 -o $O/ens_exact -f python bench.py --workload ens512_exact --steps 1 --warmup 0 --rk4-steps 20 --no-cpu-baseline > $O/ncu_exact.log 2>&1; tail -1 $O/ncu_exact.log
