"""Ensemble (DMMA GEMM, tolerance path) deviation from the pinned oracle vs horizon
('plus a reported deviation curve vs horizon').  Max |GPU - oracle| over
the recorded states of several members, recorded every H/10 steps."""
import os, sys, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_01121_b200 as sto
from oracle import oracle

n, B = int(sys.argv[1]) if len(sys.argv) > 1 else 100, 16
top = sto.build_topology(n, seed=0)
params = [sto.PhysicalParams(current=c) for c in np.linspace(2.0e-3, 3.0e-3, B)]
series = sto.InputSeries(np.random.default_rng(1).uniform(-1, 1, (10000, 1)), 1)
print(f"N={n} B={B} random drive; max over members 0, 5, 10, 15 of max |dev| over the records")
for H in [100, 300, 1000, 3000, 10000]:
    cfg = sto.RunConfig(n=n, steps=H, dt=1e-11, record_stride=max(1, H // 10),
                        input_series=sto.InputSeries(series.samples[:H], 1))
    ens = sto.integrate_ensemble(top, params, cfg)
    worst = 0.0
    for b in (0, 5, 10, 15):
        want, _ = oracle.integrate(top.coupling.entries, top.input_weights.entries,
                                   sto.kernel_scalars(params[b]), sto.initial_state(n),
                                   series.samples[:H], 1, 1e-11, H, max(1, H // 10))
        worst = max(worst, float(np.abs(ens.states[:, b] - want).max()))
    print(f"  horizon {H:6d} steps: {worst:.3e}")
