#!/bin/bash
# call ab: tiny kernel proof check every G steps (G = 1, 2, 4 default, 8): n1 bench A/B; tiny parity
mkdir -p gpurun_out/ab
O=gpurun_out/ab
for r in 1 2; do for v in G1 G2 C G8; do lib=libsto_b200_$v.so; [ $v = C ] && lib=libsto_b200.so
  STO_LIB=$lib timeout 300 python bench.py --workload n1 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', '%.5g'%d['value'], 'ms/step %.3f'%d['ms_per_step'], d['clocks']['sm_mhz'])"; done; done | tee $O/ab_n1.txt
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_division.py -m gpu -q -x -rf > $O/tests.log 2>&1; tail -2 $O/tests.log
