"""Streaming kernel near the L2 capacity: W = 8 N^2 bytes around 60-120 MB, with
the L2-resident slice budget STO_L2_KEEP_MB set by the caller.  Prints
osc-steps/s from CUDA-event kernel time (tools/l2_keep_sweep.sh companion)."""
import os, sys, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_01121_b200 as sto
from paper_2312_01121_b200 import _native
from paper_2312_01121_b200.backends.b200 import B200Backend

for n in [int(v) for v in sys.argv[1:]] or [2800, 3200, 3600, 4000]:
    g = np.random.default_rng(n)
    w = g.uniform(-1, 1, (n, n)) / np.sqrt(n / 3.0)
    np.fill_diagonal(w, 0.0)
    top = sto.Topology(sto.CouplingMatrix(w), sto.InputWeights(g.uniform(-1, 1, (n, 1))))
    be = B200Backend(top, sto.PhysicalParams(), flags=_native.FORCE_STREAM)
    cfg = sto.RunConfig(n=n, steps=2000, dt=1e-11, record_stride=2000)
    sto.integrate(top, sto.PhysicalParams(), cfg, backend=be)
    ts = []
    for _ in range(3):
        sto.integrate(top, sto.PhysicalParams(), cfg, backend=be)
        ts.append(be.last_kernel_seconds)
    t = min(ts)
    print(f"n={n} W={8*n*n/1e6:.0f} MB keep_mb={os.environ.get('STO_L2_KEEP_MB','default')} "
          f"{n*2000/t:.4g} osc-steps/s  {32.0*n*n*2000/t/1e9:.0f} GB/s-equivalent")
    be.close()
