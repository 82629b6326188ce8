#!/bin/bash
# DRAM bytes (read + write) per launch of the persistent kernel of each workload,
# for profiles/ncu_traffic.json (bench.py roofline.traffic).
mkdir -p gpurun_out
run() {  # workload rk4_steps kernel_regex
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:$3 -c 1 --csv \
      --log-file gpurun_out/traffic_$1.csv python bench.py --workload $1 --steps 1 --warmup 0 \
      --rk4-steps $2 --no-cpu-baseline > /dev/null 2>&1
}
run n1e4 20 grid_rk4
run n4e4 4 grid_rk4
run n1000 2000 reg_rk4
run ens512 200 ens_rk4
run n100 2000 clu_
run n1 20000 tiny_rk4
run ens512_exact 40 ens_exact
ls -la gpurun_out/traffic_*.csv
