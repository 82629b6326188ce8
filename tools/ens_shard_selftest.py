"""Batch-sharded ensemble check (tests/test_gpu_sharded.py): torchrun W ranks on
cuda:0 (gloo).  Every rank calls integrate_ensemble(group="world") on 13 members
(DMMA and exact mode)
(ragged split); rank 0 compares the gathered grid with the one-GPU ensemble of
all members bit for bit, and checks that a divergent member raises the same
IntegrationDivergedError (member, oscillator, step) on every rank."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_01121_b200 as sto  # noqa: E402


def main():
    dist.init_process_group("gloo")
    torch.cuda.set_device(0)
    n, steps, batch = 200, 30, 13
    top = sto.build_topology(n, seed=3)
    params = [sto.PhysicalParams(current=float(c)) for c in np.linspace(2e-3, 3e-3, batch)]
    cfg = sto.RunConfig(n=n, steps=steps, dt=1e-11, record_stride=10)
    got = sto.integrate_ensemble(top, params, cfg, group="world")
    gotx = sto.integrate_ensemble(top, params, cfg, group="world", exact=True)  # bit-exact mode
    bad = list(params)
    bad[9] = sto.PhysicalParams(h_appl=1e300)  # blows up: member 9 only (rank 1)
    try:
        sto.integrate_ensemble(top, bad, cfg, group="world")
        div = None
    except sto.IntegrationDivergedError as e:
        div = (getattr(e, "member", None), e.oscillator, e.step)
    divs = [None] * dist.get_world_size()
    dist.all_gather_object(divs, div)
    if dist.get_rank() == 0:
        want = sto.integrate_ensemble(top, params, cfg)
        try:
            sto.integrate_ensemble(top, bad, cfg)
            want_div = None
        except sto.IntegrationDivergedError as e:
            want_div = (getattr(e, "member", None), e.oscillator, e.step)
        wantx = sto.integrate_ensemble(top, params, cfg, exact=True)
        ok = bool(np.array_equal(got.states.view(np.uint64), want.states.view(np.uint64))
                  and np.array_equal(gotx.states.view(np.uint64), wantx.states.view(np.uint64))
                  and want_div is not None and all(d == want_div for d in divs))
        print(json.dumps({"ok": ok, "world": dist.get_world_size(), "divs": divs,
                          "want_div": want_div}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
