mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 | tee gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
for w in n1e4 n1 n100 n1000 ens512; do
  timeout 300 python bench.py --workload $w --steps 3 --warmup 3 > gpurun_out/q_$w.json 2> gpurun_out/q_$w.err || tail -5 gpurun_out/q_$w.err
  python -c "
import json; d=json.load(open('gpurun_out/q_$w.json'))
print('$w', '%.4g osc-steps/s'%d['value'], 'e2e %.4g'%d['e2e']['value'], 'ms/run=%.4g'%d['ms_per_step'], 'frac=%.3f'%d['roofline']['frac'], d['config'].get('kernel'), d['clocks'])"
done
