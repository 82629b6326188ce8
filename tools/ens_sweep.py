"""Ensemble throughput vs batch size at N = 1000 (tile height chosen by the host)."""
import os, sys, time, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_01121_b200 as sto
from paper_2312_01121_b200.backends.b200 import B200Backend

n = int(os.environ.get("ENS_N", 1000))
top = sto.build_topology(n, seed=0) if n <= 3000 else None
if top is None:
    g = np.random.default_rng(0); w = g.uniform(-1, 1, (n, n)) / np.sqrt(n / 3.0); np.fill_diagonal(w, 0)
    top = sto.Topology(sto.CouplingMatrix(w), sto.InputWeights(g.uniform(-1, 1, (n, 1))))
be = B200Backend(top, sto.PhysicalParams())
for B in [int(v) for v in sys.argv[1:]] or [64, 128, 256, 512, 1024, 2048]:
    consts = np.array([sto.kernel_scalars(sto.PhysicalParams(current=c)) for c in np.linspace(2e-3, 3e-3, B)])
    steps = 2000
    m0 = np.tile(sto.initial_state(n)[None], (B, 1, 1))
    be.integrate_ensemble_run(consts, np.zeros((1, 1)), 1, 1e-11, steps, steps, m0.copy())
    t = min((be.integrate_ensemble_run(consts, np.zeros((1, 1)), 1, 1e-11, steps, steps, m0.copy()),
             be.last_kernel_seconds)[1] for _ in range(2))
    rate = B * n * steps / t
    print(f"N={n} B={B:5d} {rate:.4g} osc-steps/s  {rate * 8 * n / 1e12:5.1f} TFLOP/s  {rate * 8 * n / 1e12 / 37.1:.3f} of DMMA")
