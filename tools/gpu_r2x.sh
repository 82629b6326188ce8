#!/bin/bash
# call x: configs[4] at its full benched horizon, bit-exact; long fuzz campaign (10x examples)
mkdir -p gpurun_out/x
O=gpurun_out/x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -k "benched_config4" --durations=3 > $O/config4.log 2>&1; tail -4 $O/config4.log
STO_FUZZ_SCALE=10 timeout 3000 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_ensemble.py tests/test_gpu_ensemble_exact.py tests/test_gpu_sharded.py -m gpu -q -rf -k "random" --durations=10 > $O/fuzz.log 2>&1; tail -14 $O/fuzz.log
