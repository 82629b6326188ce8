"""Row-sharded protocol on one GPU: `world` logical ranks in one launch.

Each row's tree stays on one rank, so the sharded trajectory must equal the
pinned oracle (and the unsharded kernels) bit for bit.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import assert_bit_equal, fuzz_examples

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,world,fam,chunk", [(1000, 2, 0, 0), (1000, 3, 0x1, 0), (3001, 4, 0x1, 0),
                                               (10000, 2, 0, 0), (257, 8, 0, 0),
                                               (5000, 2, 0x1, 2048), (5000, 4, 0x1, 1024),
                                               (3001, 3, 0x1, 512)])
def test_logical_ranks_bit_exact(oracle_mod, monkeypatch, n, world, fam, chunk):
    """chunk > 0: every rank's streaming kernel stages x in windows of `chunk`
    columns (STO_CHUNK_COLS), the chunked MULTI path."""
    import paper_2312_01121_b200 as sto
    from paper_2312_01121_b200.sharding import integrate_logical

    if chunk:
        monkeypatch.setenv("STO_CHUNK_COLS", str(chunk))

    g = np.random.default_rng(n + world)
    w = g.uniform(-1, 1, (n, n)) / np.sqrt(n / 3.0)
    np.fill_diagonal(w, 0.0)
    top = sto.Topology(sto.CouplingMatrix(w), sto.InputWeights(g.uniform(-1, 1, (n, 1))))
    steps = 3 if n >= 10000 else 40
    stride = max(1, steps // 4)
    samples = g.uniform(-1, 1, (steps, 1))
    consts = sto.kernel_scalars(sto.PhysicalParams())
    want, _ = oracle_mod.integrate(w, top.input_weights.entries, consts, sto.initial_state(n),
                                   samples, 1, 1e-11, steps, stride)
    m = sto.initial_state(n)
    got = integrate_logical(top, sto.PhysicalParams(), m, samples, 1, 1e-11, steps, stride,
                            world, flags=fam)
    assert_bit_equal(got, want, f"n={n} world={world}")
    assert_bit_equal(m, want[-1], "final m")


@pytest.mark.parametrize("fam", [0, 0x1])
def test_logical_ranks_multichannel_held_drive(oracle_mod, fam):
    """Sharded rows with n_in = 3 and a held drive (each rank's W_in shard, the
    input field's tree over channels, the sample index): bit-exact."""
    import paper_2312_01121_b200 as sto
    from paper_2312_01121_b200.sharding import integrate_logical

    n, world, n_in, sps, steps = 1500, 3, 3, 4, 38
    g = np.random.default_rng(77)
    w = g.uniform(-1, 1, (n, n)) / np.sqrt(n / 3.0)
    np.fill_diagonal(w, 0.0)
    w_in = g.uniform(-1, 1, (n, n_in))
    top = sto.Topology(sto.CouplingMatrix(w), sto.InputWeights(w_in))
    samples = g.uniform(-1, 1, ((steps + sps - 1) // sps, n_in))
    consts = sto.kernel_scalars(sto.PhysicalParams())
    want, _ = oracle_mod.integrate(w, w_in, consts, sto.initial_state(n), samples, sps, 1e-11,
                                   steps, 6)
    m = sto.initial_state(n)
    got = integrate_logical(top, sto.PhysicalParams(), m, samples, sps, 1e-11, steps, 6, world,
                            flags=fam)
    assert_bit_equal(got, want, "n_in=3 held drive, 3 logical ranks")


def test_repeated_group_runs_reuse_epochs(oracle_mod):
    """Epochs continue across launches (flags are never reset); two runs in a row."""
    import paper_2312_01121_b200 as sto
    from paper_2312_01121_b200 import _native
    from paper_2312_01121_b200.sharding import _shard_plan, shard_rows
    import torch

    n, world = 600, 2
    top = sto.build_topology(n, seed=3)
    consts = sto.kernel_scalars(sto.PhysicalParams())
    plans = [_shard_plan(top, consts, b, c, world, r, 0) for r, (b, c) in enumerate(shard_rows(n, world))]
    _native.connect_local(plans)
    want, _ = oracle_mod.integrate(top.coupling.entries, top.input_weights.entries, consts,
                                   sto.initial_state(n), np.zeros((1, 1)), 1, 1e-11, 30, 10)
    for _ in range(2):
        m = torch.as_tensor(sto.initial_state(n), device="cuda")
        st = torch.empty((4, n, 3), dtype=torch.float64, device="cuda")
        _native.integrate_group(plans, m, torch.zeros((1, 1), dtype=torch.float64, device="cuda"),
                                1, 1e-11, 30, 10, st)
        assert_bit_equal(st.cpu().numpy(), want)
    for p in plans:
        p.close()


def test_group_divergence_is_consistent():
    import paper_2312_01121_b200 as sto
    from paper_2312_01121_b200.sharding import integrate_logical

    n = 1200
    top = sto.Topology(sto.CouplingMatrix.zeros(n), sto.InputWeights(np.full((n, 1), 0.5)))
    drive = np.zeros((20, 1))
    drive[11:] = 1e12
    with pytest.raises(sto.IntegrationDivergedError) as info:
        integrate_logical(top, sto.PhysicalParams(), sto.initial_state(n), drive, 5, 1e-11, 100,
                          10, world=3)
    assert info.value.step == 60


@pytest.mark.parametrize("world,n", [(2, 1500), (4, 3000)])
def test_ipc_transport_multiprocess(world, n):
    """The real multi-process transport (CUDA-IPC handle exchange over
    torch.distributed, peer stores into every rank's receive buffer,
    st.release.sys epoch flags, epochs carried across runs): `world` processes
    on ONE GPU via torchrun, bit-exact against the oracle (tools/ipc_selftest.py)."""
    import json
    import socket
    import subprocess
    import sys

    from conftest import ROOT

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node",
           str(world), "--master-addr", "127.0.0.1", "--master-port", str(port),
           str(ROOT / "tools" / "ipc_selftest.py"), str(n), "2"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=240, cwd=ROOT)
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert out.returncode == 0 and lines, out.stdout[-2000:] + out.stderr[-2000:]
    res = json.loads(lines[-1])
    assert res["ok"] and res["world"] == world, res


@pytest.mark.parametrize("workload", ["n1e4", "ens512"])
def test_bench_multirank_path_on_one_gpu(workload):
    """`bench.py --gpus 2` with no external torchrun (it spawns its own ranks;
    STO_BENCH_SHARE_GPU puts both on cuda:0 with gloo): the row-sharded n1e4
    path -- ShardedB200Backend construction, IPC connect, timed runs,
    max-over-ranks, e2e with the device-side gather -- and the batch-sharded
    ensemble through integrate_ensemble(group=), each printing one valid line
    with n_gpus == 2."""
    import json
    import os
    import subprocess
    import sys

    from conftest import ROOT

    env = dict(os.environ, STO_BENCH_SHARE_GPU="1")
    env.pop("WORLD_SIZE", None)
    cmd = [sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--workload", workload,
           "--steps", "1", "--warmup", "1", "--rk4-steps", "4", "--no-cpu-baseline"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert out.returncode == 0 and len(lines) == 1, out.stdout[-2000:] + out.stderr[-3000:]
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["e2e"]["value"] > 0
    want = "row-sharded" if workload == "n1e4" else "batch-sharded"
    assert want in line["config"]["parallelism"]


def test_sharded_ensemble_matches_single_gpu():
    """integrate_ensemble(group=) over 2 ranks (torchrun, both on cuda:0, gloo)
    returns every member on every rank, bit-identical to the one-GPU ensemble
    of the same members (members are independent; the same kernel runs them)."""
    import json
    import socket
    import subprocess
    import sys

    from conftest import ROOT

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           str(ROOT / "tools" / "ens_shard_selftest.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert out.returncode == 0 and lines, out.stdout[-2000:] + out.stderr[-3000:]
    res = json.loads(lines[-1])
    assert res["ok"], res


from hypothesis import HealthCheck, given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402


@settings(max_examples=fuzz_examples(40), deadline=None, suppress_health_check=[HealthCheck.too_slow,
                                                                 HealthCheck.function_scoped_fixture])
@given(n=st.integers(8, 2500), world=st.integers(2, 8), steps=st.integers(1, 30),
       sps=st.integers(1, 5), fam=st.sampled_from([0, 0x1, 0x2 | 0x8]),
       seed=st.integers(0, 2**31 - 1))
def test_random_logical_rank_runs_bit_exact(oracle_mod, n, world, steps, sps, fam, seed):
    """Hypothesis-drawn sharded runs (world 2-8 logical ranks, ragged shards, held
    drives, streaming / SMEM-resident families): bit-exact vs the oracle."""
    import paper_2312_01121_b200 as sto
    from paper_2312_01121_b200.sharding import integrate_logical

    if n < world:
        return
    g = np.random.default_rng(seed)
    w = g.uniform(-1, 1, (n, n)) / np.sqrt(n / 3.0)
    np.fill_diagonal(w, 0.0)
    top = sto.Topology(sto.CouplingMatrix(w), sto.InputWeights(g.uniform(-1, 1, (n, 1))))
    stride = int(g.integers(1, steps + 1))
    samples = g.uniform(-1, 1, (-(-steps // sps), 1))
    consts = sto.kernel_scalars(sto.PhysicalParams())
    want, _ = oracle_mod.integrate(w, top.input_weights.entries, consts, sto.initial_state(n),
                                   samples, sps, 1e-11, steps, stride)
    m = sto.initial_state(n)
    try:
        got = integrate_logical(top, sto.PhysicalParams(), m, samples, sps, 1e-11, steps, stride,
                                world, flags=fam)
    except sto.ParameterError:
        return  # family does not fit this shard (e.g. SMEM-resident rows too wide)
    assert_bit_equal(got, want, f"n={n} world={world} fam={fam}")


def test_lost_peer_watchdog(monkeypatch):
    """A rank whose peer never launches must not hang its GPU: the exchange
    watchdog (STO_PEER_TIMEOUT_S) stops the persistent kernel and the run
    raises SpinoscError; the plan then refuses further runs (its epochs are out
    of step with the peer's)."""
    import time

    import torch

    import paper_2312_01121_b200 as sto
    from paper_2312_01121_b200 import _native
    from paper_2312_01121_b200.sharding import _shard_plan, shard_rows

    monkeypatch.setenv("STO_PEER_TIMEOUT_S", "1")
    n, world = 600, 2
    top = sto.build_topology(n, seed=5)
    consts = sto.kernel_scalars(sto.PhysicalParams())
    plans = [_shard_plan(top, consts, b, c, world, r, 0) for r, (b, c) in enumerate(shard_rows(n, world))]
    _native.connect_local(plans)
    m = torch.as_tensor(sto.initial_state(n), device="cuda")
    drive = torch.zeros((1, 1), dtype=torch.float64, device="cuda")
    st = torch.empty((2, n, 3), dtype=torch.float64, device="cuda")
    t0 = time.time()
    with pytest.raises(sto.SpinoscError, match="did not reach"):
        plans[0].integrate_dev(m, drive, 1, 1e-11, 20, 20, st)  # rank 1 never runs
    assert time.time() - t0 < 30
    with pytest.raises(sto.SpinoscError, match="lost a peer"):
        plans[0].integrate_dev(m, drive, 1, 1e-11, 20, 20, st)
    torch.cuda.synchronize()  # the device is still healthy
    for p in plans:
        p.close()
