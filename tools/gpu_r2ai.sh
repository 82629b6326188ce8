#!/bin/bash
# call ai: DMMA ensemble U x 2 tiles / split-K 4 (NT2, NT2E1 = epilogue unroll 1) vs U x 1 (C)
mkdir -p gpurun_out/ai
O=gpurun_out/ai
for r in 1 2; do for v in NT2 NT2E1 C; do lib=libsto_b200_$v.so; [ $v = C ] && lib=libsto_b200.so
  STO_LIB=$lib timeout 600 python bench.py --workload ens512 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', '%.4g'%d['value'], 'frac %.3f'%d['roofline']['frac'], d['clocks']['sm_mhz'])"; done; done | tee $O/ab.txt
STO_LIB=libsto_b200_NT2E1.so timeout 900 python -m pytest tests/test_gpu_ensemble.py -m gpu -q -x -rf > $O/tests_nt2e1.log 2>&1; tail -2 $O/tests_nt2e1.log
