#!/bin/bash
# last call of the session: full GPU suite, smoke, default bench, reference arm on the final code
mkdir -p gpurun_out/last
O=gpurun_out/last
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=10 > $O/gpu_tests.log 2>&1; tail -3 $O/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
python -c "
import json; d=json.load(open('$O/bench_default.json')); r=json.load(open('$O/bench_ref.json')); print('default', '%.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'], 'frac %.3f'%d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'], 'ref %.4g'%r['value'], 'e2e/ref %.1f'%(d['e2e']['value']/r['value']))"
for w in n1 ens512; do timeout 600 python bench.py --workload $w --no-cpu-baseline > $O/bench_$w.json 2> $O/bench_$w.err; python -c "
import json; d=json.load(open('$O/bench_$w.json')); print('$w', '%.4g'%d['value'], 'frac %.3f'%d['roofline']['frac'], d['clocks']['sm_mhz'])"; done
