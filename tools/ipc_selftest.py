"""Multi-process check of the row-sharded transport on ONE GPU (tests/test_gpu_sharded.py).

Launched as `torchrun --nproc-per-node W tools/ipc_selftest.py N STEPS`: every rank is
its own process on cuda:0 (gloo for the handle exchange), so the CUDA-IPC handle
export/import, the peer stores into every rank's receive buffer and the
st.release.sys epoch flags are exercised across process boundaries exactly as on
an NVLink box -- only the link is local.  Concurrent persistent kernels from
different processes progress by context time-slicing, so keep STEPS small.
Rank 0 prints one JSON line {"ok": bool, "max_dev": ...} comparing the assembled
trajectory with the pinned CPU oracle bit for bit.
"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_01121_b200 as sto  # noqa: E402
from paper_2312_01121_b200.sharding import ShardedB200Backend  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1500
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    dist.init_process_group("gloo")
    torch.cuda.set_device(0)
    g = np.random.default_rng(n)
    w = g.uniform(-1, 1, (n, n)) / np.sqrt(n / 3.0)
    np.fill_diagonal(w, 0.0)
    top = sto.Topology(sto.CouplingMatrix(w), sto.InputWeights(g.uniform(-1, 1, (n, 1))))
    params = sto.PhysicalParams()
    series = sto.InputSeries(g.uniform(-1, 1, (steps, 1)), 1)
    be = ShardedB200Backend(top, params, device=0)
    m = sto.initial_state(n)
    states = be.integrate_run(m, series.samples, 1, 1e-11, steps, 1)
    states2 = be.integrate_run(sto.initial_state(n), series.samples, 1, 1e-11, steps, 1)  # epochs carry over
    # a divergence on the LAST rank's rows: every rank must raise the same error
    # (the peers stop on the flag's divergence bit and learn the report through
    # agree_status) instead of the peers blocking in the state gather
    bad = sto.initial_state(n)
    bad[n - 2, 1] = np.nan
    try:
        be.integrate_run(bad, series.samples, 1, 1e-11, steps, 1)
        div = None
    except sto.IntegrationDivergedError as e:
        div = (e.oscillator, e.step)
    divs = [None] * dist.get_world_size()
    dist.all_gather_object(divs, div)
    states3 = be.integrate_run(sto.initial_state(n), series.samples, 1, 1e-11, steps, 1)  # still in step
    be.close()
    if dist.get_rank() == 0:
        from oracle import oracle

        want, _ = oracle.integrate(w, top.input_weights.entries, sto.kernel_scalars(params),
                                   sto.initial_state(n), series.samples, 1, 1e-11, steps, 1)
        try:
            oracle.integrate(w, top.input_weights.entries, sto.kernel_scalars(params), bad,
                             series.samples, 1, 1e-11, steps, 1)
            want_div = None
        except oracle.OracleDiverged as e:
            want_div = (e.oscillator, e.step)
        ok = bool(np.array_equal(states.view(np.uint64), want.view(np.uint64)) and
                  np.array_equal(states2.view(np.uint64), want.view(np.uint64)) and
                  np.array_equal(states3.view(np.uint64), want.view(np.uint64)) and
                  all(d == want_div for d in divs))
        print(json.dumps({"ok": ok, "world": dist.get_world_size(), "n": n, "steps": steps, "divergence_reports": divs,
                          "max_dev": float(np.abs(states - want).max())}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
