"""Row-sharded single trajectory over several B200s.

The reference has no multi-GPU path (`SPEC.md:349` lists it as a
non-goal); this is the B200 design for N >= 1e4: rank r owns the contiguous
oscillator rows `shard_rows(n, world)[r]` with its own slice of W; after
every RK stage the persistent kernel of each GPU stores its rows' x straight
into every peer's receive buffer over NVLink (CUDA-IPC mapped) and raises an
epoch flag there -- an all-gather of 8N bytes per stage fused into the
time-loop kernel, no NCCL call per stage (see csrc/sto_kernels.cuh,
`multi_sync`). Each row's tree sum stays on one rank, so results are
bit-identical to the unsharded run.

Two front ends share the same kernel and protocol:

* `ShardedB200Backend`: one process per GPU under torch.distributed
  (torchrun). Plans exchange 64-byte IPC handles with `all_gather_object`;
  `integrate_run` returns the full recorded grid on every rank.
* `integrate_logical`: `world` logical ranks on ONE GPU in one launch
  (plain device buffers instead of IPC peers) -- how the exchange protocol is
  exercised on a single-GPU box.
"""

from __future__ import annotations

import numpy as np

from . import _native
from .errors import ParameterError
from .params import kernel_scalars


def shard_rows(n: int, world: int) -> list[tuple[int, int]]:
    """Contiguous balanced row blocks [(row_begin, row_count)] for `world` ranks."""
    if world < 1 or n < world:
        raise ParameterError(f"cannot shard {n} rows over {world} ranks")
    bounds = [(r * n) // world for r in range(world + 1)]
    return [(bounds[r], bounds[r + 1] - bounds[r]) for r in range(world)]


def assemble_states(blocks: list[np.ndarray], shards: list[tuple[int, int]], n: int) -> np.ndarray:
    """Full (R, n, 3) grid from each rank's (R, rows_r, 3) block."""
    nrec = blocks[0].shape[0]
    out = np.empty((nrec, n, 3))
    for (begin, count), blk in zip(shards, blocks):
        if blk.shape != (nrec, count, 3):
            raise ParameterError("state block does not match its shard")
        out[:, begin:begin + count] = blk
    return out


def _shard_plan(topology, consts, begin: int, count: int, world: int, rank: int, device: int,
                flags: int = 0) -> _native.Plan:
    w = topology.coupling.entries[begin:begin + count]
    w_in = topology.input_weights.entries[begin:begin + count]
    return _native.Plan(w, w_in, consts, device=device, flags=flags,
                        shard=(begin, count, world, rank))


def integrate_logical(topology, params, m0: np.ndarray, samples: np.ndarray,
                      steps_per_sample: int, dt: float, steps: int, stride: int, world: int,
                      device: int = 0, flags: int = 0, consts=None) -> np.ndarray:
    """Run the sharded protocol with `world` logical ranks on one GPU.

    Returns the recorded states (R, n, 3); m0 is updated in place."""
    import torch

    n = topology.n
    consts = kernel_scalars(params) if consts is None else consts
    shards = shard_rows(n, world)
    plans = [_shard_plan(topology, consts, b, c, world, r, device, flags)
             for r, (b, c) in enumerate(shards)]
    try:
        _native.connect_local(plans)
        dev = torch.device("cuda", device)
        m_d = torch.as_tensor(np.ascontiguousarray(m0, dtype=np.float64)).to(dev)
        s_d = torch.as_tensor(np.ascontiguousarray(samples, dtype=np.float64)).to(dev)
        states = torch.empty((_native.n_records(steps, stride), n, 3), dtype=torch.float64,
                             device=dev)
        _native.integrate_group(plans, m_d, s_d, steps_per_sample, dt, steps, stride, states)
        np.copyto(m0, m_d.cpu().numpy())
        return states.cpu().numpy()
    finally:
        for p in plans:
            p.close()


class ShardedB200Backend:
    """One rank of a row-sharded trajectory (one process per GPU, torch.distributed).

    Collective construction: every rank of the default process group must
    create it with the same topology and parameters.
    """

    backend_id = "gpu"
    kind = "B200 persistent RK4, row-sharded over NVLink"

    def __init__(self, topology, params, device: int | None = None, group=None, flags: int = 0):
        import torch
        import torch.distributed as dist

        self._dist, self._group, self._torch = dist, group, torch
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.n = topology.n
        self.shards = shard_rows(self.n, self.world)
        begin, count = self.shards[self.rank]
        self._plan = _shard_plan(topology, kernel_scalars(params), begin, count, self.world,
                                 self.rank, self.device, flags)
        handles: list = [None] * self.world
        dist.all_gather_object(handles, self._plan.exchange_handle(), group=group)
        self._plan.connect(handles)
        dist.barrier(group=group)

    def integrate_run(self, m0: np.ndarray, samples: np.ndarray, steps_per_sample: int,
                      dt: float, steps: int, stride: int) -> np.ndarray:
        torch, dist = self._torch, self._dist
        dev = torch.device("cuda", self.device)
        begin, count = self.shards[self.rank]
        m_d = torch.as_tensor(np.ascontiguousarray(m0, dtype=np.float64)).to(dev)
        s_d = torch.as_tensor(np.ascontiguousarray(samples, dtype=np.float64)).to(dev)
        nrec = _native.n_records(steps, stride)
        states = torch.zeros((nrec, self.n, 3), dtype=torch.float64, device=dev)
        dist.barrier(group=self._group)  # nobody starts before every peer finished the last run
        self._plan.integrate_dev(m_d, s_d, steps_per_sample, dt, steps, stride, states, sync=True)
        mine = states[:, begin:begin + count].cpu().numpy()
        blocks: list = [None] * self.world
        dist.all_gather_object(blocks, (mine, m_d[begin:begin + count].cpu().numpy()),
                               group=self._group)
        full = assemble_states([b[0] for b in blocks], self.shards, self.n)
        for (b, c), blk in zip(self.shards, blocks):
            m0[b:b + c] = blk[1]
        return full

    def close(self) -> None:
        self._plan.close()
