"""Cluster kernel (csrc/sto_cluster_kernel.cuh) vs the register kernel for small N:
bit-exact check against the oracle on a short recorded run with a drive, then
RK4 steps/s over a long run, for every (cluster size K, columns per thread C)."""
import os, sys, numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2312_01121_b200 import _native as nat
if os.environ.get("STO_LIB"):  # A/B builds
    nat.LIB_PATH = nat.LIB_PATH.with_name(os.environ["STO_LIB"])
import paper_2312_01121_b200 as sto
from paper_2312_01121_b200 import _native as nat
from paper_2312_01121_b200.backends.b200 import B200Backend
from oracle import oracle

oracle.build()
ns = [int(v) for v in sys.argv[1:]] or [33, 64, 100, 128, 200, 256]
n_in = int(os.environ.get("N_IN", "1"))
for n in ns:
    g = np.random.default_rng(n)
    w = g.uniform(-1, 1, (n, n)) / np.sqrt(n / 3.0)
    np.fill_diagonal(w, 0.0)
    w_in = g.uniform(-1, 1, (n, n_in))
    top = sto.Topology(sto.CouplingMatrix(w), sto.InputWeights(w_in))
    params = sto.PhysicalParams()
    m0 = sto.initial_state(n)
    samples = g.uniform(-1, 1, (19, n_in))
    want, _ = oracle.integrate(w, w_in, sto.kernel_scalars(params), m0, samples, 3, 1e-11, 57, 4)
    variants = [("reg", nat.FORCE_REG | nat.NO_TINY, {})]
    for hyb in (1, 0):
        for c in (64, 32, 16):
            for k in (2, 4, 8, 16):
                variants.append((f"{'hyb' if hyb else 'own'} K={k} C={c}", nat.FORCE_CLUSTER,
                                 {"STO_CLU_K": str(k), "STO_CLU_C": str(c), "STO_CLU_HYB": str(hyb)}))
    for name, flags, env in variants:
        for key in ("STO_CLU_K", "STO_CLU_C", "STO_CLU_HYB"):
            os.environ.pop(key, None)
        os.environ.update(env)
        try:
            be = B200Backend(top, params, flags=flags)
        except Exception as exc:
            print(f"n={n:4d} {name:14s} -- {str(exc)[:60]}")
            continue
        m = m0.copy()
        got = be.integrate_run(m, samples, 3, 1e-11, 57, 4)
        ok = np.array_equal(got.view(np.uint64), want.view(np.uint64))
        steps = 20000
        drive = g.uniform(-1, 1, (steps, n_in))  # a new sample every step (bench n100)
        ts = []
        for _ in range(3):
            be.integrate_run(m0.copy(), drive, 1, 1e-11, steps, steps)
            ts.append(be.last_kernel_seconds)
        t = min(ts)
        info = be.plan_info
        print(f"n={n:4d} {name:14s} grid={info['grid']:3d} thr={info['threads']:4d} "
              f"{'BITEXACT' if ok else 'MISMATCH'} {steps/t:.4g} steps/s {t/steps*1e9:7.1f} ns/step "
              f"{n*steps/t:.4g} osc-steps/s", flush=True)
        be.close()
