#!/bin/bash
# call u: DMMA ensemble with readiness-ordered K loop (tests + bench x2)
mkdir -p gpurun_out/u
O=gpurun_out/u
timeout 1200 python -m pytest tests/test_gpu_ensemble.py -m gpu -q -x -rf > $O/tests.log 2>&1; tail -3 $O/tests.log
for r in 1 2; do timeout 900 python bench.py --workload ens512 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_ens512_$r.json 2> $O/bench_ens512_$r.err; python -c "
import json; d=json.loads(open('$O/bench_ens512_$r.json').read()); print('ens512', '%.4g'%d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'])"; done
