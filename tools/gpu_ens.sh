#!/bin/bash
# ensemble kernel: parity tests, bench line, per-phase timeline (debug build)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ensemble.py -x -q 2>&1 | tail -15
python bench.py --workload ens512 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/q_ens512.json 2> gpurun_out/q_ens512.err || tail -5 gpurun_out/q_ens512.err
python -c "
import json; d=json.load(open('gpurun_out/q_ens512.json'))
print('ens512', '%.4g osc-steps/s'%d['value'], 'ms/run=%.4g'%d['ms_per_step'], 'frac=%.3f'%d['roofline']['frac'], d['clocks'])"
make -C paper_2312_01121_b200/csrc timeline -s > /dev/null 2>&1 && timeout 300 python tools/ens_timeline.py 2>&1 | tail -8
