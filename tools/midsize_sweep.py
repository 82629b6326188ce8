"""Throughput of the automatically chosen kernel across mid-size N (the reference's
FULL_GRID has 2500 / 5000 / 10000): osc-steps/s and W-bytes-equivalent GB/s."""
import os, sys, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_01121_b200 as sto
from paper_2312_01121_b200.backends.b200 import B200Backend

for n in [int(v) for v in sys.argv[1:]] or [1200, 1500, 2000, 2500, 3500, 5000, 7000]:
    g = np.random.default_rng(n)
    w = g.uniform(-1, 1, (n, n)) / np.sqrt(n / 3.0)
    np.fill_diagonal(w, 0.0)
    top = sto.Topology(sto.CouplingMatrix(w), sto.InputWeights(g.uniform(-1, 1, (n, 1))))
    be = B200Backend(top, sto.PhysicalParams())
    steps = max(200, int(4e9 / (32.0 * n * n)))
    cfg = sto.RunConfig(n=n, steps=steps, dt=1e-11, record_stride=steps)
    sto.integrate(top, sto.PhysicalParams(), cfg, backend=be)
    t = min(sto.integrate(top, sto.PhysicalParams(), cfg, backend=be) and be.last_kernel_seconds for _ in range(3))
    info = be.plan_info
    print(f"n={n:5d} kernel={info['kernel_name']:9s} grid={info['grid']:3d} W={8*n*n/1e6:6.1f} MB "
          f"{n*steps/t:.4g} osc-steps/s  {32.0*n*n*steps/t/1e9:6.0f} GB/s-eq  {t/steps/4*1e6:6.2f} us/stage")
    be.close()
