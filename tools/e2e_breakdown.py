"""Where the e2e time of a large-N run goes (bench.py e2e path): pinned-host W
-> plan creation (H2D + permute) -> integrate -> read-back.  python
tools/e2e_breakdown.py N STEPS"""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2312_01121_b200 as sto
from paper_2312_01121_b200.backends.b200 import B200Backend

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 40000
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
top_d = sto.build_topology_device(n, seed=0)
w_pin = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
t0 = time.perf_counter(); w_pin.copy_(top_d.coupling.tensor); torch.cuda.synchronize()
d2h = time.perf_counter() - t0
x = torch.empty((n, n), dtype=torch.float64, device="cuda")
t0 = time.perf_counter(); x.copy_(w_pin); torch.cuda.synchronize()
h2d = time.perf_counter() - t0
print(f"pinned D2H {8*n*n/d2h/1e9:.1f} GB/s, H2D {8*n*n/h2d/1e9:.1f} GB/s ({h2d*1e3:.0f} ms)")
del x, top_d
torch.cuda.empty_cache()
top = sto.Topology(sto.CouplingMatrix(w_pin.numpy()), sto.InputWeights(np.full((n, 1), 0.5)))
params = sto.PhysicalParams()
cfg = sto.RunConfig(n=n, steps=steps, dt=1e-11, record_stride=steps)
for rep in range(3):
    t0 = time.perf_counter(); be = B200Backend(top, params); torch.cuda.synchronize(); t1 = time.perf_counter()
    tr = sto.integrate(top, params, cfg, backend=be); t2 = time.perf_counter()
    be.close(); t3 = time.perf_counter()
    tot = time.perf_counter()
    t4 = time.perf_counter(); tr2 = sto.integrate(top, params, cfg); t5 = time.perf_counter()
    print(f"plan {1e3*(t1-t0):.0f} ms, integrate {1e3*(t2-t1):.0f} ms (kernel {1e3*be.last_kernel_seconds:.0f}), "
          f"close {1e3*(t3-t2):.0f} ms; public integrate() end to end {1e3*(t5-t4):.0f} ms")
