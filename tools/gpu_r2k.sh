#!/bin/bash
# round 2 session 3, first call: full GPU suite, smoke, every bench workload, reference arm,
# launch list of the default bench, compute-sanitizer over every kernel family
mkdir -p gpurun_out/k
O=gpurun_out/k
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/nvsmi.txt
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=20 > $O/gpu_tests.log 2>&1; tail -5 $O/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -2 $O/smoke.log
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; cat $O/bench_default.json
for w in n1 n100 n100_rec1 n1000 ens512 n4e4 n1e4_rec10; do
  timeout 900 python bench.py --workload $w > $O/bench_$w.json 2> $O/bench_$w.err; head -c 300 $O/bench_$w.json; echo
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_default.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
SAN_TIMEOUT=240 timeout 3000 bash tools/sanitize.sh memcheck synccheck racecheck > /dev/null 2>&1
cp -r gpurun_out/sanitize $O/ 2>/dev/null; cat $O/sanitize/summary.txt | cut -c1-150
