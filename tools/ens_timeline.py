"""Per-phase cycle timeline of the ensemble kernel (debug build)."""
import ctypes, sys
import numpy as np
sys.path.insert(0, ".")
import paper_2312_01121_b200._native as nat
nat.LIB_PATH = nat.LIB_PATH.with_name("libsto_b200_timeline.so")
import paper_2312_01121_b200 as sto

n, B = 1000, 512
top = sto.build_topology(n, seed=0) if len(sys.argv) < 2 else None
if top is None:
    g = np.random.default_rng(0); w = g.uniform(-1, 1, (n, n)) / 18.0; np.fill_diagonal(w, 0)
    top = sto.Topology(sto.CouplingMatrix(w), sto.InputWeights(g.uniform(-1, 1, (n, 1))))
params = [sto.PhysicalParams(current=c) for c in np.linspace(2e-3, 3e-3, B)]
cfg = sto.RunConfig(n=n, steps=30, dt=1e-11, record_stride=30)
sto.integrate_ensemble(top, params, cfg)
buf = (ctypes.c_ulonglong * 128)()
nat.lib().sto_debug_ens_timeline(buf, 128)
t = np.array(buf, dtype=np.float64).reshape(16, 2, 4)
t0 = t[0, 0, 0]
for s in range(15):
    line = f"stage {40+s}:"
    for g in range(2):
        gemm, epi, total = t[s, g, 1] - t[s, g, 0], t[s, g, 2] - t[s, g, 1], t[s + 1, g, 0] - t[s, g, 0]
        line += (f" | g{g} start {t[s, g, 0] - t0:8.0f} gemm {gemm:6.0f} (data wait {t[s, g, 3]:6.0f}) epi {epi:6.0f}"
                 f" exch {total - gemm - epi:6.0f} total {total:6.0f}")
    print(line)
