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

from paper_2312_01121_b200.sharding import assemble_states, shard_rows


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
