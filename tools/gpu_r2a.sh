#!/bin/bash
# round 2 first call: full GPU suite (incl. the chunked-x / full-horizon tests), smoke, default bench
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=15 2>&1 | tail -40 | tee gpurun_out/a_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee gpurun_out/a_smoke.log
python bench.py > gpurun_out/a_default.json 2> gpurun_out/a_default.err; cat gpurun_out/a_default.json
