"""Per-phase cycles of the grid kernel, CTA 0 (debug build libsto_b200_timeline.so):
python tools/grid_timeline.py N [flags]"""
import ctypes, sys
import numpy as np
sys.path.insert(0, ".")
import paper_2312_01121_b200._native as nat
nat.LIB_PATH = nat.LIB_PATH.with_name("libsto_b200_timeline.so")
import paper_2312_01121_b200 as sto
from paper_2312_01121_b200.backends.b200 import B200Backend

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
flags = int(sys.argv[2], 0) if len(sys.argv) > 2 else 0
g = np.random.default_rng(0)
w = g.uniform(-1, 1, (n, n)) / np.sqrt(n); np.fill_diagonal(w, 0)
top = sto.Topology(sto.CouplingMatrix(w), sto.InputWeights(g.uniform(-1, 1, (n, 1))))
be = B200Backend(top, sto.PhysicalParams(), flags=flags)
print(be.plan_info)
m = sto.initial_state(n)
be.integrate_run(m, np.zeros((1, 1)), 1, 1e-11, 40, 40)
buf = (ctypes.c_ulonglong * 80)()
L = ctypes.CDLL(str(nat.LIB_PATH))
L.sto_debug_grid_timeline(buf, 80)
t = np.array(buf, dtype=np.float64).reshape(16, 5)
for s in range(15):
    d = np.diff(t[s])
    print(f"stage {100+s}: x-stage {d[0]:6.0f}  block {d[1]:6.0f}  rows {d[2]:6.0f}  barrier {d[3]:6.0f}  total {t[s+1,0]-t[s,0]:6.0f} cyc")

cb = (ctypes.c_ulonglong * 2048)()
L.sto_debug_grid_cta_block(cb, 2048)
a = np.array(cb, dtype=np.float64).reshape(2, 1024)[:, :be.plan_info["grid"]]
start, end = a[0] - a[0].min(), a[1] - a[0].min()
dur = a[1] - a[0]
print(f"stage 100 block phase per CTA (globaltimer ns): start spread {start.max():.0f}, "
      f"duration min {dur.min():.0f} median {np.median(dur):.0f} max {dur.max():.0f}, "
      f"end spread {end.max() - end.min():.0f}")
print("slowest CTAs:", np.argsort(-dur)[:8].tolist(), "fastest:", np.argsort(dur)[:8].tolist())
