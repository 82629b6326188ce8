#!/bin/bash
# One GPU session: bench lines for every workload + ncu launch list + full capture.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python bench.py --steps 3 --warmup 3 > gpurun_out/bench_n1e4.json 2> gpurun_out/bench_n1e4.err; tail -3 gpurun_out/bench_n1e4.err
cat gpurun_out/bench_n1e4.json
for w in n1000 n100 n1; do
  python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; tail -2 gpurun_out/bench_$w.err
  cat gpurun_out/bench_$w.json
done
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref_n1e4.json 2>&1; cat gpurun_out/ref_n1e4.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_n1e4.csv python bench.py --steps 2 --warmup 1 --rk4-steps 20 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:grid_rk4 -c 1 -o gpurun_out/prof_n1e4 -f python bench.py --steps 1 --warmup 0 --rk4-steps 10 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; tail -3 gpurun_out/ncu_full.log
ls -la gpurun_out
