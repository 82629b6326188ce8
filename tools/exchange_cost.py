"""Per-RK-stage cost of the row-sharded exchange, measured with logical ranks on
one GPU: the same MULTI grid kernel and protocol as the
multi-GPU path (each CTA pushes its x slice into every rank's receive buffer,
local counter barrier, epoch flags with st.release.sys, fence.acq_rel.sys),
only the peer buffers are local.  world = 1 is the unsharded grid kernel
(grid barrier, no peer stores).  Every plan streams W (FORCE_STREAM), so the
CTA-level work is the same and the difference is the exchange.  Prints one JSON line per (n, world):
microseconds per RK stage and the difference to world = 1.

    python tools/exchange_cost.py [n ...]
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2312_01121_b200 as sto  # noqa: E402
from paper_2312_01121_b200 import _native  # noqa: E402
from paper_2312_01121_b200.sharding import _shard_plan, shard_rows  # noqa: E402


def topo(n):
    g = np.random.default_rng(n)
    w = g.uniform(-1, 1, (n, n)) / np.sqrt(n / 3.0)
    np.fill_diagonal(w, 0.0)
    return sto.Topology(sto.CouplingMatrix(w), sto.InputWeights(g.uniform(-1, 1, (n, 1))))


def time_runs(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(reps):
        a.record()
        fn()
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b) / 1e3)
    return best


def main():
    sizes = [int(float(v)) for v in sys.argv[1:]] or [2000, 10000]
    consts = sto.kernel_scalars(sto.PhysicalParams())
    for n in sizes:
        steps = max(200, int(4e9 / (32.0 * n * n)))
        top = topo(n)
        u = torch.zeros((1, 1), dtype=torch.float64, device="cuda")
        base = None
        for world in (1, 2, 4, 8):
            m0 = torch.as_tensor(sto.initial_state(n), device="cuda")
            m = m0.clone()
            if world == 1:
                plan = _native.Plan(top.coupling.entries, top.input_weights.entries, consts,
                                    device=0, flags=_native.FORCE_STREAM)
                kind = plan.info["kernel_name"]

                def run():
                    m.copy_(m0)
                    plan.integrate_dev(m, u, 1, 1e-11, steps, steps, None)
                plans = [plan]
            else:
                plans = [_shard_plan(top, consts, b, c, world, r, 0, _native.FORCE_STREAM)
                         for r, (b, c) in enumerate(shard_rows(n, world))]
                _native.connect_local(plans)
                kind = "MULTI"

                def run():
                    m.copy_(m0)
                    _native.integrate_group(plans, m, u, 1, 1e-11, steps, steps, None)
            sec = time_runs(run)
            us = sec / (4 * steps) * 1e6
            if base is None:
                base = us
            print(json.dumps({"n": n, "world": world, "kernel": str(kind), "steps": steps,
                              "us_per_stage": round(us, 3),
                              "exchange_over_unsharded_us": round(us - base, 3)}), flush=True)
            for p in plans:
                p.close()


if __name__ == "__main__":
    main()
