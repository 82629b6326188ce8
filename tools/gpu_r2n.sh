#!/bin/bash
# call n: ncu --set full of the exact and DMMA ensemble kernels; exchange cost; n1 bench
mkdir -p gpurun_out/n
O=gpurun_out/n
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ens_exact -c 1 -o $O/ens_exact -f python bench.py --workload ens512_exact --steps 1 --warmup 0 --rk4-steps 20 --no-cpu-baseline > $O/ncu_exact.log 2>&1; tail -2 $O/ncu_exact.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ens_rk4 -c 1 -o $O/ens_dmma -f python bench.py --workload ens512 --steps 1 --warmup 0 --rk4-steps 20 --no-cpu-baseline > $O/ncu_dmma.log 2>&1; tail -2 $O/ncu_dmma.log
timeout 600 python tools/exchange_cost.py 2000 10000 > $O/exchange_cost.jsonl 2> $O/exchange_cost.err; cat $O/exchange_cost.jsonl; tail -2 $O/exchange_cost.err
timeout 600 python bench.py --workload n1 > $O/bench_n1.json 2> $O/bench_n1.err; head -c 300 $O/bench_n1.json
