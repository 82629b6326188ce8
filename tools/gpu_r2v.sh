#!/bin/bash
# call v: device norm drift + pinned D2H (tests, e2e of dense recording); sanitizers on the kernels changed this round
mkdir -p gpurun_out/v
O=gpurun_out/v
timeout 1500 python -m pytest tests/test_gpu_drift.py tests/test_gpu_parity.py tests/test_gpu_ensemble.py tests/test_gpu_sharded.py -m gpu -q -x -rf > $O/tests.log 2>&1; tail -3 $O/tests.log
for w in n100_rec1 n1e4_rec10 n100; do timeout 900 python bench.py --workload $w --no-cpu-baseline > $O/bench_$w.json 2> $O/bench_$w.err; python -c "
import json; d=json.loads(open('$O/bench_$w.json').read()); print('$w', '%.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'], d['clocks']['sm_mhz'])"; done
CASES="tiny_n7 tiny_n1_spec multi_w2_n600 multi_w4_n1500_chunked ensemble_u7 ensemble_exact cluster_hyb_k8_n100_div" SAN_TIMEOUT=300 timeout 2400 bash tools/sanitize.sh memcheck synccheck racecheck > /dev/null 2>&1; cp -r gpurun_out/sanitize $O/; cut -c1-160 $O/sanitize/summary.txt
