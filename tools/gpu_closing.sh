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
# ncu evidence of the N = 100 cluster kernel (clu_hyb_kernel) and the default launch list
ncu --set full --clock-control none --import-source on -k regex:clu_ -c 1 -o gpurun_out/c_clu_n100 -f python bench.py --workload n100 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/c_clu_ncu.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c_launches_default.csv python bench.py --steps 2 --warmup 1 --rk4-steps 50 --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c_launches_n100.csv python bench.py --workload n100 --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out/c_*
