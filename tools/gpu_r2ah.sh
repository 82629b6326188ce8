#!/bin/bash
# call ah: DMMA ensemble with alternating GEMM turns (C) vs free-running groups (A0): tests, A/B bench
mkdir -p gpurun_out/ah
O=gpurun_out/ah
timeout 1200 python -m pytest tests/test_gpu_ensemble.py -m gpu -q -x -rf > $O/tests.log 2>&1; tail -2 $O/tests.log
for r in 1 2; do for v in A0 C; do lib=libsto_b200_$v.so; [ $v = C ] && lib=libsto_b200.so
  STO_LIB=$lib timeout 600 python bench.py --workload ens512 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', '%.4g'%d['value'], 'frac %.3f'%d['roofline']['frac'], d['clocks']['sm_mhz'])"; done; done | tee $O/ab.txt
