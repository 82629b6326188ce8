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
from .errors import IntegrationDivergedError, ParameterError, SpinoscError
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


# status words agreed across ranks after every sharded run (agree_status)
RUN_OK, RUN_DIVERGED, RUN_FAILED = 0, 1, 2


def collective_device(group=None):
    """Device of the tensors a collective on `group` takes: the current CUDA
    device under NCCL, the host under gloo (CPU tests, STO_BENCH_SHARE_GPU)."""
    import torch
    import torch.distributed as dist

    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def agree_status(status: tuple[int, int, int], group=None,
                 local_error: Exception | None = None) -> None:
    """Every rank raises the same error after a sharded run, or none does.

    `status` = (RUN_*, oscillator, step) of this rank's launch.  A divergence
    is detected by the rank owning the bad row only; its peers learn of it
    through the divergence bit of that epoch's exchange flag and stop cleanly
    at the same epoch with an OK status.  Without this exchange the owning
    rank would raise while its peers went on into the state gather and
    blocked forever.  The earliest (step, oscillator) over the diverged ranks
    is the reference's report (integrator.py:174-177: first bad recorded step,
    first bad row in it); a watchdog stop or CUDA error on any rank becomes a
    SpinoscError on every rank."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    mine = torch.tensor([int(v) for v in status], dtype=torch.int64,
                        device=collective_device(group))
    every = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(every, mine, group=group)
    rows = [tuple(int(v) for v in t.cpu().tolist()) for t in every]
    failed = [r for r, s in enumerate(rows) if s[0] == RUN_FAILED]
    if failed:
        why = f": {local_error}" if local_error is not None else "; see that rank's error"
        raise SpinoscError(f"sharded run failed on rank(s) {failed} (peer watchdog or CUDA "
                           f"error){why}") from local_error
    bad = [(s[2], s[1]) for s in rows if s[0] == RUN_DIVERGED]
    if bad:
        step, osc = min(bad)
        raise IntegrationDivergedError(oscillator=osc, step=step)


def gather_rows(block, shards: list[tuple[int, int]], n: int, group=None):
    """All-gather row blocks into the full array on every rank.

    `block` is this rank's (R, rows_r, 3) slice of a row-sharded array (a
    torch tensor on `collective_device(group)`); returns the (R, n, 3) tensor
    with every rank's rows in place.  Device-side under NCCL: one padded
    all_gather over NVLink instead of pickling every rank's states."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rows_max = max(c for _, c in shards)
    rank = dist.get_rank(group)
    if block.shape[1] != shards[rank][1]:
        raise ParameterError("row block does not match this rank's shard")
    padded = torch.zeros((block.shape[0], rows_max, *block.shape[2:]), dtype=block.dtype,
                         device=block.device)
    padded[:, :block.shape[1]] = block
    parts = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(parts, padded, group=group)
    return torch.cat([parts[r][:, :c] for r, (_, c) in enumerate(shards)], dim=1)


def shard_members(batch: int, world: int, rank: int) -> np.ndarray:
    """Member indices rank `rank` integrates when a batch of independent
    ensemble members is batch-sharded over `world` ranks (contiguous and
    balanced, so the gathered order is the member order)."""
    if world < 1 or not 0 <= rank < world:
        raise ParameterError(f"bad rank {rank} of {world}")
    return np.array_split(np.arange(batch), world)[rank]


def integrate_ensemble_sharded(backend, consts: np.ndarray, samples: np.ndarray,
                               steps_per_sample: int, config, group, exact: bool = False,
                               m0: np.ndarray | None = None) -> np.ndarray:
    """Batch-sharded ensemble: this rank's members on its own
    GPU, then one all-gather of the recorded grids.  consts (B, 11) and
    samples ([B,] n_samples, n_in) describe the WHOLE batch; returns the
    (R, B, n, 3) grid on every rank (see integrate_ensemble)."""
    import torch.distributed as dist

    from .topology import initial_state

    group = None if group == "world" else group
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    batch = consts.shape[0]
    if batch < world:
        raise ParameterError(f"cannot batch-shard {batch} members over {world} ranks")
    mine = shard_members(batch, world, rank)
    counts = [(0, len(shard_members(batch, world, r))) for r in range(world)]
    samples_mine = samples[mine] if samples.ndim == 3 else samples
    if m0 is None:
        m = np.tile(initial_state(config.n, config.phi0)[None], (len(mine), 1, 1))
    else:
        m = np.ascontiguousarray(m0[mine])
    local_error = None
    states = None
    try:
        states = backend.integrate_ensemble_run(consts[mine], samples_mine, steps_per_sample,
                                                config.dt, config.steps, config.record_stride, m,
                                                exact=exact)
        status = (RUN_OK, 0, 0)
    except IntegrationDivergedError as exc:
        # step, then global member, then oscillator: packed so min() keeps that order
        member = int(mine[0]) + int(getattr(exc, "member", 0))
        status = (RUN_DIVERGED, member * (1 << 32) + exc.oscillator, exc.step)
    except SpinoscError as exc:
        status, local_error = (RUN_FAILED, 0, 0), exc
    try:
        agree_status(status, group, local_error)
    except IntegrationDivergedError as exc:
        err = IntegrationDivergedError(oscillator=exc.oscillator & 0xffffffff, step=exc.step)
        err.member = exc.oscillator >> 32
        raise err from None
    import torch

    block = torch.as_tensor(states).to(collective_device(group))
    return gather_rows(block, counts, batch, group).cpu().numpy()


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
        """The whole run on every rank; returns the full recorded grid (R, n, 3)
        on every rank and updates m0 (n, 3) in place.  A divergence raises
        IntegrationDivergedError on every rank (agree_status)."""
        torch, dist = self._torch, self._dist
        dev = torch.device("cuda", self.device)
        begin, count = self.shards[self.rank]
        m_d = torch.as_tensor(np.ascontiguousarray(m0, dtype=np.float64)).to(dev)
        s_d = torch.as_tensor(np.ascontiguousarray(samples, dtype=np.float64)).to(dev)
        nrec = _native.n_records(steps, stride)
        states = torch.zeros((nrec + 1, self.n, 3), dtype=torch.float64, device=dev)
        dist.barrier(group=self._group)  # nobody starts before every peer finished the last run
        local_error = None
        try:
            self._plan.integrate_dev(m_d, s_d, steps_per_sample, dt, steps, stride, states,
                                     sync=True)
            status = (RUN_OK, 0, 0)
        except IntegrationDivergedError as exc:
            status = (RUN_DIVERGED, exc.oscillator, exc.step)
        except SpinoscError as exc:
            status, local_error = (RUN_FAILED, 0, 0), exc
        agree_status(status, self._group, local_error)
        # final state rides along as one more "record" of this rank's rows
        states[nrec, begin:begin + count] = m_d[begin:begin + count]
        block = states[:, begin:begin + count].to(collective_device(self._group))
        full = gather_rows(block, self.shards, self.n, self._group).cpu().numpy()
        np.copyto(m0, full[nrec])
        return full[:nrec]

    def close(self) -> None:
        self._plan.close()
