"""A/B of library builds (STO_LIB=<file in paper_2312_01121_b200/>) on the
automatically selected kernel: bit-exact check against the oracle on a short
recorded run with a drive, then RK4 steps/s over a long run.
Usage: STO_LIB=libsto_b200_x.so python tools/lib_ab.py N [N ...]"""
import os, sys, numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2312_01121_b200 import _native as nat
if os.environ.get("STO_LIB"):
    nat.LIB_PATH = nat.LIB_PATH.with_name(os.environ["STO_LIB"])
import paper_2312_01121_b200 as sto
from paper_2312_01121_b200.backends.b200 import B200Backend
from oracle import oracle

oracle.build()
for n in [int(v) for v in sys.argv[1:]] or [1000]:
    g = np.random.default_rng(n)
    w = g.uniform(-1, 1, (n, n)) / np.sqrt(n / 3.0)
    np.fill_diagonal(w, 0.0)
    w_in = g.uniform(-1, 1, (n, 1))
    top = sto.Topology(sto.CouplingMatrix(w), sto.InputWeights(w_in))
    params = sto.PhysicalParams()
    m0 = sto.initial_state(n)
    samples = g.uniform(-1, 1, (19, 1))
    want, _ = oracle.integrate(w, w_in, sto.kernel_scalars(params), m0, samples, 3, 1e-11, 57, 4)
    be = B200Backend(top, params)
    got = be.integrate_run(m0.copy(), samples, 3, 1e-11, 57, 4)
    ok = np.array_equal(got.view(np.uint64), want.view(np.uint64))
    steps = 20000
    ts = []
    for _ in range(3):
        be.integrate_run(m0.copy(), np.zeros((1, 1)), 1, 1e-11, steps, steps)
        ts.append(be.last_kernel_seconds)
    t = min(ts)
    print(f"{os.environ.get('STO_LIB', 'default'):28s} n={n:5d} {be.plan_info['kernel_name']:8s} "
          f"{'BITEXACT' if ok else 'MISMATCH'} {t/steps*1e9:7.1f} ns/step {n*steps/t:.4g} osc-steps/s", flush=True)
    be.close()
