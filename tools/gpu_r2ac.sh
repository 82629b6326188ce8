#!/bin/bash
# call ac: four-DFMA speculative division (STO_DIV_SHORT=1) vs default: proof rate, chain, n1
mkdir -p gpurun_out/ac
O=gpurun_out/ac
./tools/microbench_d4 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('D4 ddiv_spec', d['ddiv_spec_cyc'], 'rk4_spec', d['rk4_step_spec_cyc'], 'replays', d['rk4_spec_replays'])"
STO_LIB=libsto_b200_D4.so timeout 600 python -m pytest tests/test_gpu_division.py -m gpu -q -rf > $O/div_d4.log 2>&1; tail -3 $O/div_d4.log
STO_LIB=libsto_b200_D4.so python - <<'PY'
import numpy as np, torch, sys
sys.path.insert(0, ".")
from paper_2312_01121_b200 import _native
g = np.random.default_rng(0)
for name, a, b in [("rhs", np.full(4_000_000, 134.86812645902467), 1 + 0.288 * g.uniform(-1.5, 1.5, 4_000_000)),
                   ("wide", g.uniform(1, 2, 4_000_000) * np.exp2(g.integers(-300, 300, 4_000_000)), g.uniform(1, 2, 4_000_000) * np.exp2(g.integers(-150, 150, 4_000_000)))]:
    q, ok, ref = _native.selftest_div(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda())
    ok = ok.cpu().numpy().astype(bool); q = q.cpu().numpy(); ref = ref.cpu().numpy()
    print(name, "proved fraction", ok.mean(), "proved-but-wrong", int((ok & (q.view(np.uint64) != ref.view(np.uint64))).sum()), "unproved-but-right", int((~ok & (q.view(np.uint64) == ref.view(np.uint64))).sum()))
PY
for r in 1 2; do for v in D4 C; do lib=libsto_b200_$v.so; [ $v = C ] && lib=libsto_b200.so
  STO_LIB=$lib timeout 300 python bench.py --workload n1 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', '%.5g'%d['value'], 'ms/step %.3f'%d['ms_per_step'], d['clocks']['sm_mhz'])"; done; done
STO_LIB=libsto_b200_D4.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -q -x -rf > $O/parity_d4.log 2>&1; tail -2 $O/parity_d4.log
