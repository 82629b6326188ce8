#!/bin/bash
# round 2 call b: new/changed GPU tests, ensemble horizon bar
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_ensemble.py tests/test_gpu_parity.py -m gpu -q -x -rf -s -k "bench_multirank or sharded_ensemble or ipc or benched_config or full_horizon or llg_derivative or derivative" 2>&1 | tail -30 > gpurun_out/b2_tests.log
timeout 900 python tools/ens_horizon_bar.py 0,511 > gpurun_out/ens_bar.json 2> gpurun_out/ens_bar.err
