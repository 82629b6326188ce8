#!/bin/bash
# round 2 call c: cluster-kernel changes (relaxed wait, record flags on the mbarrier)
mkdir -p gpurun_out
for c in cluster_hyb_k8_n100_div cluster_own_k16_n200_div cluster_hyb_k2_n50 cluster_c64_n400; do timeout 120 python tools/sanitize_case.py $c 2>&1 | tail -1; done > gpurun_out/c2_cases.log
timeout 1200 python -m pytest tests -m gpu -q -x -rf -k "cluster or golden or fuzz or parity_sizes or resume" 2>&1 | tail -15 > gpurun_out/c2_tests.log
for w in n100 n100_rec1 n1e4_rec10; do timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c2_$w.json 2> gpurun_out/c2_$w.err; done
timeout 900 python tools/clu_sweep.py 64 100 128 200 256 > gpurun_out/c2_clu_sweep.log 2>&1
