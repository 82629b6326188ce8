import os, sys, numpy as np
sys.path.insert(0, ".")
import paper_2312_01121_b200 as sto
from paper_2312_01121_b200.backends.b200 import B200Backend
n = int(sys.argv[1])
g = np.random.default_rng(n)
w = g.uniform(-1, 1, (n, n)) / np.sqrt(n / 3.0); np.fill_diagonal(w, 0.0)
top = sto.Topology(sto.CouplingMatrix(w), sto.InputWeights(g.uniform(-1, 1, (n, 1))))
be = B200Backend(top, sto.PhysicalParams())
cfg = sto.RunConfig(n=n, steps=100, dt=1e-11, record_stride=100)
sto.integrate(top, sto.PhysicalParams(), cfg, backend=be)
