#!/bin/bash
# call ae: ncu --set full of the latency-bound kernels on the final code (n1 tiny, n100 cluster, n1000 reg);
# summaries made on the box (the reports are too large to bring back together)
mkdir -p gpurun_out/ae
O=gpurun_out/ae
R=/tmp/ncu_ae; mkdir -p $R
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tiny_rk4 -c 1 -o $R/tiny_n1 -f python bench.py --workload n1 --steps 1 --warmup 0 --rk4-steps 20000 --no-cpu-baseline > $O/ncu_tiny.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:clu_ -c 1 -o $R/clu_n100 -f python bench.py --workload n100 --steps 1 --warmup 0 --rk4-steps 2000 --no-cpu-baseline > $O/ncu_clu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:reg_rk4 -c 1 -o $R/reg_n1000 -f python bench.py --workload n1000 --steps 1 --warmup 0 --rk4-steps 2000 --no-cpu-baseline > $O/ncu_reg.log 2>&1
python tools/ncu_summary.py $R/tiny_n1.ncu-rep $R/clu_n100.ncu-rep $R/reg_n1000.ncu-rep > $O/summary.txt 2>&1
for k in tiny_n1 clu_n100 reg_n1000; do python tools/ncu_hot.py $R/$k.ncu-rep 30 > $O/hot_$k.txt 2>&1; done
cp $R/tiny_n1.ncu-rep $O/ 2>/dev/null
cat $O/summary.txt
