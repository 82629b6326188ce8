#!/bin/bash
# streaming kernel: L2-resident W slice sweep (STO_L2_KEEP_MB), n1e4 and n4e4
for w in n1e4 n4e4; do
for mb in 0 32 48 64 80 96; do
  STO_L2_KEEP_MB=$mb python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$w keep_mb=$mb', '%.4g osc-steps/s'%d['value'], 'frac %.3f'%d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done; done
