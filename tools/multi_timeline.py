"""Per-phase cycles of the MULTI grid kernel with `world` logical ranks on one GPU
(CTA 0 of rank 0; debug build libsto_b200_timeline.so, `make -C
paper_2312_01121_b200/csrc timeline`): python tools/multi_timeline.py N WORLD
(WORLD = 1: the unsharded streaming kernel).  Phases: x staging, block phase
(W . x nodes), row phase (RHS, RK4, x push), exchange (barrier / multi_sync)."""
import ctypes, sys
import numpy as np
sys.path.insert(0, ".")
import paper_2312_01121_b200._native as nat
import os
nat.LIB_PATH = nat.LIB_PATH.with_name(os.environ.get("STO_TL_LIB", "libsto_b200_timeline.so"))
import torch
import paper_2312_01121_b200 as sto
from paper_2312_01121_b200.sharding import _shard_plan, shard_rows

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10000
world = int(sys.argv[2]) if len(sys.argv) > 2 else 2
g = np.random.default_rng(0)
w = g.uniform(-1, 1, (n, n)) / np.sqrt(n); np.fill_diagonal(w, 0)
top = sto.Topology(sto.CouplingMatrix(w), sto.InputWeights(g.uniform(-1, 1, (n, 1))))
consts = sto.kernel_scalars(sto.PhysicalParams())
u = torch.zeros((1, 1), dtype=torch.float64, device="cuda")
m = torch.as_tensor(sto.initial_state(n), device="cuda")
if world == 1:
    plan = nat.Plan(top.coupling.entries, top.input_weights.entries, consts, flags=nat.FORCE_STREAM)
    plan.integrate_dev(m, u, 1, 1e-11, 40, 40, None)
    plans = [plan]
else:
    plans = [_shard_plan(top, consts, b, c, world, r, 0, nat.FORCE_STREAM)
             for r, (b, c) in enumerate(shard_rows(n, world))]
    nat.connect_local(plans)
    nat.integrate_group(plans, m, u, 1, 1e-11, 40, 40, None)
print(plans[0].info)
buf = (ctypes.c_ulonglong * 80)()
L = ctypes.CDLL(str(nat.LIB_PATH))
L.sto_debug_grid_timeline(buf, 80)
t = np.array(buf, dtype=np.float64).reshape(16, 5)
rows = []
for s in range(15):
    d = np.diff(t[s])
    rows.append(list(d) + [t[s + 1, 0] - t[s, 0]])
    print(f"stage {100+s}: x-stage {d[0]:7.0f}  block {d[1]:7.0f}  rows {d[2]:7.0f}  exchange {d[3]:7.0f}  "
          f"total {t[s+1,0]-t[s,0]:7.0f} cyc")
med = np.median(np.array(rows), axis=0)
print(f"median: x-stage {med[0]:.0f} block {med[1]:.0f} rows {med[2]:.0f} exchange {med[3]:.0f} total {med[4]:.0f} cyc")
if world > 1:
    mb = (ctypes.c_ulonglong * 80)()
    L.sto_debug_multi_timeline(mb, 80)
    mt = np.array(mb, dtype=np.float64).reshape(16, 5)
    d = np.median(np.diff(mt[:15], axis=1), axis=0)
    print(f"multi_sync median: own fence {d[0]:.0f}  local barrier {d[1]:.0f}  flags {d[2]:.0f}  "
          f"acquire fence {d[3]:.0f} cyc")
