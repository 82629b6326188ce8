#!/bin/bash
mkdir -p gpurun_out
for c in cluster_hyb_k8_n100_div cluster_own_k16_n200_div; do timeout 120 python tools/sanitize_case.py $c 2>&1 | tail -1; done > gpurun_out/d2_cases.log
for w in n100 n100_rec1 n100 n100_rec1; do timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline 2> /dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$w', '%.4g'%d['value'], 'ms/step %.3f'%d['ms_per_step'], 'e2e %.4g'%d['e2e']['value'], d['clocks']['sm_mhz'])"; done > gpurun_out/d2_bench.log 2>&1
