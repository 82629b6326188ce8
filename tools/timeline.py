"""Per-phase timeline of the reg kernel (debug build libsto_b200_timeline.so)."""
import ctypes, sys
import numpy as np
sys.path.insert(0, ".")
import paper_2312_01121_b200._native as nat
import os
nat.LIB_PATH = nat.LIB_PATH.with_name(os.environ.get("STO_LIB", "libsto_b200_timeline.so"))
import paper_2312_01121_b200 as sto
from paper_2312_01121_b200.backends.b200 import B200Backend

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
g = np.random.default_rng(0)
w = g.uniform(-1, 1, (n, n)) / np.sqrt(n); np.fill_diagonal(w, 0)
top = sto.Topology(sto.CouplingMatrix(w), sto.InputWeights(g.uniform(-1, 1, (n, 1))))
be = B200Backend(top, sto.PhysicalParams())
print(be.plan_info)
m = sto.initial_state(n)
be.integrate_run(m, np.zeros((1, 1)), 1, 1e-11, 200, 200)
be.integrate_run(m, np.zeros((1, 1)), 1, 1e-11, 200, 200)
buf = (ctypes.c_ulonglong * (2 * 16 * 5))()
nat.lib().sto_debug_timeline(buf, 2 * 16 * 5)
t = np.array(buf, dtype=np.float64).reshape(2, 16, 5)
t0 = t[0, 0, 0]
names = ["start", "gemv+sync", "rhs+store", "ll read", "sync"]
for who in range(2):
    print("CTA", "first" if who == 0 else "last")
    for s in range(16):
        row = t[who, s] - t0
        d = np.diff(t[who, s])
        if be.plan_info["kernel_name"] == "cluster" and os.environ.get("STO_CLU_HYB", "1") != "0" and n <= 128:
            # clu_hyb_kernel: 3 team got x, 4 butterfly done, 1 RHS post + update done, 2 published
            nx = t[who, s + 1] if s < 15 else t[who, s] * np.nan
            print(f"  stage {400+s}: cycle {nx[3] - t[who, s, 3]:6.0f}  gemv {t[who, s, 4] - t[who, s, 3]:5.0f}  "
                  f"post {t[who, s, 1] - t[who, s, 4]:5.0f}  publish {t[who, s, 2] - t[who, s, 1]:5.0f}  "
                  f"exchange {nx[3] - t[who, s, 2]:6.0f}")
            continue
        if be.plan_info["kernel_name"] == "cluster":
            # events: 0 owner has row sums, 1 post+update done, 2 published,
            #         3 GEMV warp got x, 4 GEMV butterfly done
            nx = t[who, s + 1] if s < 15 else t[who, s] * np.nan
            print(f"  stage {400+s}: cycle {nx[0] - t[who, s, 0]:6.0f}  post {d[0]:5.0f}  publish {d[1]:5.0f}  "
                  f"exchange {nx[3] - t[who, s, 2]:6.0f}  gemv {nx[4] - nx[3]:5.0f}  handoff {nx[0] - nx[4]:5.0f}")
            continue
        print(f"  stage {400+s}: start {row[0]:8.0f} cyc gemv {d[0]:6.0f}  rhs {d[1]:6.0f}  ll {d[2]:6.0f}  sync {d[3]:6.0f}  total->{(t[who, s+1, 0] - t[who, s, 0]) if s < 15 else 0:6.0f}")
