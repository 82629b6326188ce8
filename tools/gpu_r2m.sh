#!/bin/bash
# call m: bit-exact ensemble mode (tests, bench, sanitizer), ensemble DMMA changes, microbench
mkdir -p gpurun_out/m
O=gpurun_out/m
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -std=c++17 -I paper_2312_01121_b200/csrc tools/microbench.cu -o tools/microbench 2>/dev/null && ./tools/microbench > $O/microbench.json; cat $O/microbench.json
timeout 1500 python -m pytest tests/test_gpu_ensemble_exact.py tests/test_gpu_ensemble.py -m gpu -q -x -rf --durations=10 > $O/tests.log 2>&1; tail -15 $O/tests.log
timeout 900 python bench.py --workload ens512_exact --steps 3 --warmup 3 > $O/bench_ens512_exact.json 2> $O/bench_ens512_exact.err; head -c 1500 $O/bench_ens512_exact.json; tail -3 $O/bench_ens512_exact.err
CASES="ensemble_exact ensemble_exact_2launch ensemble_u1" SAN_TIMEOUT=300 timeout 1500 bash tools/sanitize.sh memcheck synccheck racecheck > /dev/null 2>&1; cp -r gpurun_out/sanitize $O/; cat $O/sanitize/summary.txt | cut -c1-200
