"""One logical-rank MULTI run (for ncu): python tools/multi_run.py N WORLD STEPS"""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2312_01121_b200 as sto
from paper_2312_01121_b200 import _native as nat
from paper_2312_01121_b200.sharding import integrate_logical

n, world, steps = int(float(sys.argv[1])), int(sys.argv[2]), int(sys.argv[3])
g = np.random.default_rng(0)
w = g.uniform(-1, 1, (n, n)) / np.sqrt(n); np.fill_diagonal(w, 0)
top = sto.Topology(sto.CouplingMatrix(w), sto.InputWeights(g.uniform(-1, 1, (n, 1))))
m = sto.initial_state(n)
integrate_logical(top, sto.PhysicalParams(), m, np.zeros((1, 1)), 1, 1e-11, steps, steps, world,
                  flags=nat.FORCE_STREAM)
print("ok")
