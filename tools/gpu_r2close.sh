#!/bin/bash
# round-2 closing run: full GPU suite, smoke, both bench arms, every workload, launch list
# and one ncu --set full capture of the default bench's kernel.  $1 = output tag
T=${1:-z}
O=gpurun_out/close_$T
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/nvsmi.txt
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=20 > $O/gpu_tests.log 2>&1; tail -3 $O/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; head -c 400 $O/bench_default.json; echo
for w in n1 n100 n100_rec1 n1000 ens512 ens512_exact n4e4 n1e4_rec10; do
  timeout 900 python bench.py --workload $w > $O/bench_$w.json 2> $O/bench_$w.err
  python -c "
import json; d=json.loads(open('$O/bench_$w.json').read()); print('$w', '%.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'], 'frac %.3f'%d['roofline']['frac'], d['clocks']['sm_mhz'])" 2>&1 | tail -1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_default.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:grid_rk4 -c 1 -o $O/stream_n1e4 -f python bench.py --steps 1 --warmup 0 --rk4-steps 20 --no-cpu-baseline > $O/ncu_stream.log 2>&1; tail -1 $O/ncu_stream.log
