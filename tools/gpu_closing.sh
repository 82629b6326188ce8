#!/bin/bash
# closing run of a round: full GPU suite, smoke, default bench + reference arm, every workload
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 | tee gpurun_out/c_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee gpurun_out/c_smoke.log
python bench.py --impl reference > gpurun_out/c_ref.json 2> gpurun_out/c_ref.err; cat gpurun_out/c_ref.json
python bench.py > gpurun_out/c_default.json 2> gpurun_out/c_default.err; cat gpurun_out/c_default.json
for w in n1 n100 n1000 ens512 n4e4; do
  timeout 600 python bench.py --workload $w --steps 3 --warmup 3 > gpurun_out/c_$w.json 2> gpurun_out/c_$w.err || tail -3 gpurun_out/c_$w.err
  python -c "
import json; d=json.load(open('gpurun_out/c_$w.json'))
print('$w', '%.4g osc-steps/s'%d['value'], 'e2e %.4g'%d['e2e']['value'], 'frac=%.3f'%d['roofline']['frac'], d['config'].get('kernel'), 'cpu %.3g'%d['cpu_baseline']['value'], d['clocks'])"
done
