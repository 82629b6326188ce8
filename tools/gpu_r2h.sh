#!/bin/bash
mkdir -p gpurun_out
for c in cluster_hyb_k8_n100_div cluster_own_k16_n200_div cluster_hyb_k2_n50 cluster_hyb_k16_n200; do timeout 120 python tools/sanitize_case.py $c 2>&1 | tail -1; done > gpurun_out/j2_cases.log
timeout 1200 python -m pytest tests -m gpu -q -x -rf -k "cluster or golden or fuzz" 2>&1 | tail -3 >> gpurun_out/j2_cases.log
bash tools/ab_bench.sh "A C" "n100 n100_rec1" 2 > gpurun_out/ab5.log 2>&1
