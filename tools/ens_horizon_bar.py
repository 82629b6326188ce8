"""configs[3] parity bar vs horizon (VERDICT r1 'pin the ensemble'): N = 1000,
B = 512 (current sweep 2.0-3.0 mA), build_topology(1000, seed=0), u = 0.

For sampled members: max |x - oracle| over the recorded states of
  * our DMMA ensemble (integrate_ensemble, the benched path),
  * the reference's OWN GPU backend (spinosc TorchBackend from baseline/_ref,
    cuBLAS `mv` order + reciprocal-multiply division, gpu.py:83-119),
at 1e3 and 1e4 RK4 steps.  The reference holds its GPU path to 1e-10 at 1e3
steps (cli.py:227-233) and states no bar beyond; its own backend's deviation at
1e4 is the bar this prints for the benched horizon.  Writes one JSON line.
    python tools/ens_horizon_bar.py [ref_members] > gpurun_out/ens_bar.json
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2312_01121_b200 as sto  # noqa: E402
from oracle import oracle  # noqa: E402

n, B = 1000, 512
ref_members = [int(v) for v in sys.argv[1].split(",")] if len(sys.argv) > 1 else [0, 511]
ours_members = [0, 73, 146, 219, 292, 365, 438, 511]
top = sto.build_topology(n, seed=0)
currents = np.linspace(2.0e-3, 3.0e-3, B)
params = [sto.PhysicalParams(current=float(c)) for c in currents]
out = {"n": n, "batch": B, "members": ours_members, "ref_members": ref_members}

sys.path.append(os.path.join(ROOT, "baseline", "_ref"))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_sto")
import spinosc  # noqa: E402
from spinosc import topology as rtop  # noqa: E402

rtopo = rtop.Topology(rtop.CouplingMatrix(top.coupling.entries),
                      rtop.InputWeights(top.input_weights.entries))

for H in (1000, 10000):
    stride = H // 10
    cfg = sto.RunConfig(n=n, steps=H, dt=1e-11, record_stride=stride)
    t0 = time.time()
    ens = sto.integrate_ensemble(top, params, cfg)
    t_ens = time.time() - t0
    dev_ours, dev_ref, want_cache = {}, {}, {}
    for b in sorted(set(ours_members) | set(ref_members)):
        want, _ = oracle.integrate(top.coupling.entries, top.input_weights.entries,
                                   sto.kernel_scalars(params[b]), sto.initial_state(n),
                                   np.zeros((1, 1)), 1, 1e-11, H, stride)
        if b in ours_members:
            dev_ours[b] = float(np.abs(ens.states[:, b] - want).max())
        if b in ref_members:
            rp = spinosc.PhysicalParams(current=float(currents[b]))
            t1 = time.time()
            tr = spinosc.integrate(rtopo, rp, spinosc.RunConfig(n=n, steps=H, dt=1e-11,
                                                                 record_stride=stride,
                                                                 backend="gpu", gpu_device=0))
            dev_ref[b] = float(np.abs(tr.states - want).max())
            out[f"ref_seconds_H{H}_b{b}"] = time.time() - t1
    out[f"H{H}"] = {"ours_max": max(dev_ours.values()), "ours": dev_ours,
                    "ref_torch_max": max(dev_ref.values()), "ref_torch": dev_ref,
                    "ens_seconds": t_ens}
    print(H, out[f"H{H}"], file=sys.stderr, flush=True)
print(json.dumps(out), flush=True)
