import time, sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2312_01121_b200 as sto
from paper_2312_01121_b200 import _native
from paper_2312_01121_b200.backends.b200 import B200Backend
n = 10000
g = np.random.default_rng(0)
w_pin = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
w_pin.numpy()[...] = g.uniform(-1, 1, (n, n)) / 58.0
np.fill_diagonal(w_pin.numpy(), 0.0)
top = sto.Topology(sto.CouplingMatrix(w_pin.numpy()), sto.InputWeights(g.uniform(-1, 1, (n, 1))))
params = sto.PhysicalParams()
cfg = sto.RunConfig(n=n, steps=1000, dt=1e-11, record_stride=1000, backend="gpu")
sto.integrate(top, params, cfg)
for rep in range(2):
    t0 = time.perf_counter(); be = B200Backend(top, params); torch.cuda.synchronize(); t1 = time.perf_counter()
    tr = sto.integrate(top, params, cfg, backend=be); t2 = time.perf_counter()
    be.close(); t3 = time.perf_counter()
    print(f"plan create {1e3*(t1-t0):.1f} ms, integrate {1e3*(t2-t1):.1f} ms (kernel {1e3*be.last_kernel_seconds:.1f}), close {1e3*(t3-t2):.1f} ms")
t0 = time.perf_counter(); _native.probe(0); print("probe %.2f ms" % (1e3*(time.perf_counter()-t0)))
