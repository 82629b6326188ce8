#!/bin/bash
# tests + per-workload bench lines (no ncu)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
for w in ${WORKLOADS:-n1 n100 n1000 n1e4 ens512}; do
  python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/q_$w.json 2> gpurun_out/q_$w.err || tail -5 gpurun_out/q_$w.err
  python -c "
import json; d=json.load(open('gpurun_out/q_$w.json'))
print('$w', '%.4g osc-steps/s'%d['value'], 'ms/run=%.4g'%d['ms_per_step'], 'frac=%.3f'%d['roofline']['frac'], d['config']['kernel'], d['config']['grid'], d['clocks'])"
done
