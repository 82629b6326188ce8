#!/bin/bash
# call ay: DMMA ensemble epilogue unroll 1 / 2 (default C) / 4 A/B
mkdir -p gpurun_out/ay
for r in 1 2; do for v in E1 C E4; do lib=libsto_b200_$v.so; [ $v = C ] && lib=libsto_b200.so
  STO_LIB=$lib timeout 600 python bench.py --workload ens512 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', '%.4g'%d['value'], 'frac %.3f'%d['roofline']['frac'], d['clocks']['sm_mhz'])"; done; done | tee gpurun_out/ay/ab.txt
