#!/bin/bash
mkdir -p gpurun_out/ad
O=gpurun_out/ad
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -std=c++17 -I paper_2312_01121_b200/csrc tools/microbench.cu -o tools/microbench 2>/dev/null && ./tools/microbench > $O/microbench.json; python -c "import json; d=json.load(open('$O/microbench.json')); print({k:d[k] for k in ('ddiv_cyc','ddiv_spec_cyc','rk4_step_spec_cyc','rk4_spec_replays')})"
timeout 1500 python -m pytest tests/test_gpu_division.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_cluster.py -m gpu -q -x -rf > $O/tests.log 2>&1; tail -2 $O/tests.log
timeout 600 python bench.py --workload n1 > $O/bench_n1.json 2> $O/bench_n1.err; python -c "
import json; d=json.load(open('$O/bench_n1.json')); print('n1', '%.4g'%d['value'], d['roofline']['frac'], d['roofline']['peak'], d['clocks']['sm_mhz'])"
