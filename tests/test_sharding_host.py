"""Host-side logic of the row-sharded multi-GPU path, on CPU.

World-size-2 `gloo` process group: shard partition, the all-gather of IPC
exchange handles and the reassembly of per-rank state blocks, i.e. what
`ShardedB200Backend` does around the kernel.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2312_01121_b200.sharding import (RUN_DIVERGED, RUN_FAILED, RUN_OK, agree_status,
                                            assemble_states, gather_rows, shard_members,
                                            shard_rows)


@pytest.mark.parametrize("n,world", [(8, 2), (10, 3), (10000, 8), (1001, 7)])
def test_shard_rows_cover_exactly_once(n, world):
    shards = shard_rows(n, world)
    assert len(shards) == world
    assert shards[0][0] == 0
    for (b0, c0), (b1, _) in zip(shards, shards[1:]):
        assert b0 + c0 == b1
    assert shards[-1][0] + shards[-1][1] == n
    assert max(c for _, c in shards) - min(c for _, c in shards) <= 1


def test_shard_rows_rejects_too_many_ranks():
    from paper_2312_01121_b200 import ParameterError

    with pytest.raises(ParameterError):
        shard_rows(3, 4)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shards = shard_rows(n, world)
        # stand-in for sto_plan_exchange_handle: 64 opaque bytes per rank
        handle = bytes([rank]) * 64
        handles = [None] * world
        dist.all_gather_object(handles, handle)
        assert handles == [bytes([r]) * 64 for r in range(world)]
        # each rank contributes its rows of a known grid; everyone reassembles
        full = np.arange(5 * n * 3, dtype=np.float64).reshape(5, n, 3)
        begin, count = shards[rank]
        blocks = [None] * world
        dist.all_gather_object(blocks, full[:, begin:begin + count].copy())
        got = assemble_states(blocks, shards, n)
        result_q.put((rank, bool(np.array_equal(got, full))))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_handle_exchange_and_assembly():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, 37, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    results = sorted(q.get(timeout=10) for _ in procs)
    assert results == [(0, True), (1, True)]
    assert all(p.exitcode == 0 for p in procs)


def _collective_worker(rank, world, port, n, result_q):
    """gather_rows (padded device-style all_gather of ragged row blocks) and
    agree_status (every rank raises the same error) on a gloo group."""
    import torch

    from paper_2312_01121_b200 import IntegrationDivergedError, SpinoscError

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = {}
    try:
        shards = shard_rows(n, world)
        full = torch.arange(4 * n * 3, dtype=torch.float64).reshape(4, n, 3)
        begin, count = shards[rank]
        got = gather_rows(full[:, begin:begin + count].clone(), shards, n)
        out["gather"] = bool(torch.equal(got, full))
        agree_status((RUN_OK, 0, 0))  # nobody diverged: no error anywhere
        out["ok"] = True
        # ranks 1 and 2 diverge at different (step, oscillator): everyone reports the earliest
        st = {1: (RUN_DIVERGED, 7, 40), 2: (RUN_DIVERGED, 3, 20)}.get(rank, (RUN_OK, 0, 0))
        try:
            agree_status(st)
            out["div"] = None
        except IntegrationDivergedError as e:
            out["div"] = (e.oscillator, e.step)
        # a watchdog stop on one rank fails every rank, even a diverged one
        st = (RUN_FAILED, 0, 0) if rank == world - 1 else (RUN_DIVERGED, 1, 1)
        try:
            agree_status(st)
            out["fail"] = None
        except IntegrationDivergedError:
            out["fail"] = "diverged"
        except SpinoscError:
            out["fail"] = "failed"
        result_q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_gloo_world3_status_agreement_and_row_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = 3
    procs = [ctx.Process(target=_collective_worker, args=(r, world, port, 11, q))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    results = dict(q.get(timeout=10) for _ in procs)
    assert all(p.exitcode == 0 for p in procs)
    for r in range(world):
        assert results[r] == {"gather": True, "ok": True, "div": (3, 20), "fail": "failed"}, results


@pytest.mark.parametrize("batch,world", [(512, 8), (512, 3), (7, 4), (3, 3)])
def test_shard_members_partition(batch, world):
    got = np.concatenate([shard_members(batch, world, r) for r in range(world)])
    assert np.array_equal(got, np.arange(batch))
    sizes = [len(shard_members(batch, world, r)) for r in range(world)]
    assert max(sizes) - min(sizes) <= 1
