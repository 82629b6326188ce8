mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_sharded.py -x -q 2>&1 | tail -5
STO_LIB=libsto_b200_timeline.so timeout 120 python tools/timeline.py 100 2>&1 | tail -40 > gpurun_out/tl100.txt
STO_LIB=libsto_b200_timeline.so timeout 120 python tools/timeline.py 1000 2>&1 | tail -40 > gpurun_out/tl1000.txt
cat gpurun_out/tl100.txt | head -22
cat gpurun_out/tl1000.txt | head -22
