bash tools/gpu_traffic.sh > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:grid_rk4 -c 1 -o gpurun_out/j_stream_n1e4 -f python bench.py --steps 1 --warmup 0 --rk4-steps 10 --no-cpu-baseline > gpurun_out/j_ncu.log 2>&1
ls gpurun_out/traffic_*.csv gpurun_out/j_stream_n1e4.ncu-rep
