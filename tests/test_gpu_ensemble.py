"""Batched ensemble (DMMA GEMM coupling) against the pinned oracle, per member.

Bar: every member within 1e-10 absolute of the oracle run
with that member's parameters after 1e3 RK4 steps -- the reference's own
GPU tolerance (`cli.py:232`). The GEMM accumulates in tensor-core order,
not the pinned tree, so bit-equality is not expected here; the measured
deviation is printed (-s) for the record.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import fuzz_examples

pytestmark = pytest.mark.gpu

TOL = 1e-10


@pytest.fixture(scope="module")
def sto():
    import paper_2312_01121_b200 as sto

    return sto


def test_benched_config_members_within_reference_gpu_tolerance(sto, oracle_mod):
    """configs[3] exactly as benched (bench.py ens512): N = 1000, B = 512, the
    2.0-3.0 mA sweep, build_topology(1000, seed=0), u = 0; 8 members across the
    sweep, every 100th step recorded, within 1e-10 of the pinned oracle at
    1e3 RK4 steps (the reference's GPU bar, cli.py:227-233).  The benched
    horizon (1e4) is held to the reference's own GPU backend's deviation there
    (tools/ens_horizon_bar.py)."""
    n, batch, steps = 1000, 512, 1000
    top = sto.build_topology(n, seed=0)
    params = _sweep(sto, batch)
    cfg = sto.RunConfig(n=n, steps=steps, dt=1e-11, record_stride=100)
    ens = sto.integrate_ensemble(top, params, cfg)
    assert ens.states.shape == (11, batch, n, 3)
    worst = 0.0
    for b in (0, 73, 146, 219, 292, 365, 438, 511):
        want, _ = oracle_mod.integrate(top.coupling.entries, top.input_weights.entries,
                                       sto.kernel_scalars(params[b]), sto.initial_state(n),
                                       np.zeros((1, 1)), 1, 1e-11, steps, 100)
        dev = float(np.abs(ens.states[:, b] - want).max())
        worst = max(worst, dev)
        assert dev <= TOL, f"member {b}: {dev:.3e}"
    print(f"configs[3] at 1e3 steps: max deviation {worst:.3e} over 8 members")


# configs[3] at the benched horizon (1e4 RK4 steps): the reference states no
# GPU bar beyond 1e3 steps (cli.py:227-233).  Its OWN GPU backend (spinosc
# TorchBackend: cuBLAS mv order, gpu.py:83-119) deviates from the pinned CPU
# path by 7.9e-10 (member 0) / 3.7e-10 (member 511) there -- the dynamics
# amplify any rounding-order difference ~10x per 3e3 steps -- and this DMMA
# path by 1.1e-9 / 3.9e-10, max 3.4e-9 over 8 members (tools/ens_horizon_bar.py,
# profiles/r02b_ens_horizon_bar.json).  Bar at 1e4 steps: 1e-8.  (The exact
# ensemble mode is bit-identical at any horizon.)
TOL_1E4 = 1e-8


def test_benched_horizon_members_within_stated_bar(sto, oracle_mod):
    n, batch, steps = 1000, 512, 10_000
    top = sto.build_topology(n, seed=0)
    params = _sweep(sto, batch)
    cfg = sto.RunConfig(n=n, steps=steps, dt=1e-11, record_stride=1000)
    ens = sto.integrate_ensemble(top, params, cfg)
    worst = 0.0
    for b in (0, 146, 511):
        want, _ = oracle_mod.integrate(top.coupling.entries, top.input_weights.entries,
                                       sto.kernel_scalars(params[b]), sto.initial_state(n),
                                       np.zeros((1, 1)), 1, 1e-11, steps, 1000)
        dev = float(np.abs(ens.states[:, b] - want).max())
        worst = max(worst, dev)
        assert dev <= TOL_1E4, f"member {b}: {dev:.3e} at 1e4 steps"
    print(f"configs[3] at 1e4 steps: max deviation {worst:.3e} over 3 members")


def _sweep(sto, batch):
    return [sto.PhysicalParams(current=c) for c in np.linspace(2.0e-3, 3.0e-3, batch)]


@pytest.mark.parametrize("n,batch,steps", [(100, 70, 1000), (257, 16, 1000), (1000, 8, 200)])
def test_members_match_oracle(sto, oracle_mod, n, batch, steps):
    top = sto.build_topology(n, seed=n) if n <= 300 else None
    if top is None:
        g = np.random.default_rng(n)
        w = g.uniform(-1, 1, (n, n)) / np.sqrt(n / 3.0)
        np.fill_diagonal(w, 0.0)
        top = sto.Topology(sto.CouplingMatrix(w), sto.InputWeights(g.uniform(-1, 1, (n, 1))))
    params = _sweep(sto, batch)
    stride = steps // 4
    series = sto.InputSeries(np.random.default_rng(5).uniform(-1, 1, (steps, 1)), 1)
    cfg = sto.RunConfig(n=n, steps=steps, dt=1e-11, record_stride=stride, input_series=series)
    ens = sto.integrate_ensemble(top, params, cfg)
    assert ens.states.shape == (steps // stride + 1, batch, n, 3)
    worst = 0.0
    for b in range(batch) if batch <= 16 else list(range(0, batch, 7)) + [batch - 1]:
        want, _ = oracle_mod.integrate(top.coupling.entries, top.input_weights.entries,
                                       sto.kernel_scalars(params[b]), sto.initial_state(n),
                                       series.samples, 1, 1e-11, steps, stride)
        dev = float(np.abs(ens.states[:, b] - want).max())
        worst = max(worst, dev)
        assert dev <= TOL, f"member {b}: deviation {dev:.3e}"
    print(f"ensemble n={n} B={batch} steps={steps}: worst member deviation {worst:.3e}")


def test_member_view_and_drift(sto):
    top = sto.build_topology(40, seed=1)
    ens = sto.integrate_ensemble(top, _sweep(sto, 3), sto.RunConfig(n=40, steps=50, dt=1e-11,
                                                                     record_stride=10))
    tr = ens.member(2)
    assert tr.states.shape == (6, 40, 3)
    assert ens.max_norm_drift.shape == (3,)
    assert np.all(ens.max_norm_drift < 1e-6)


def test_per_member_drive(sto, oracle_mod):
    n, steps = 64, 120
    top = sto.build_topology(n, seed=2)
    g = np.random.default_rng(3)
    series = [sto.InputSeries(g.uniform(-1, 1, (40, 1)), 3) for _ in range(5)]
    params = [sto.PhysicalParams()] * 5
    ens = sto.integrate_ensemble(top, params, sto.RunConfig(n=n, steps=steps, dt=1e-11,
                                                            record_stride=40),
                                 input_series=series)
    for b in range(5):
        want, _ = oracle_mod.integrate(top.coupling.entries, top.input_weights.entries,
                                       sto.kernel_scalars(params[b]), sto.initial_state(n),
                                       series[b].samples, 3, 1e-11, steps, 40)
        assert float(np.abs(ens.states[:, b] - want).max()) <= TOL


def test_ensemble_divergence_reports_member(sto):
    n = 16
    top = sto.Topology.decoupled(n)
    params = [sto.PhysicalParams()] * 3 + [sto.PhysicalParams(h_appl=1e300)]
    with pytest.raises(sto.IntegrationDivergedError) as info:
        sto.integrate_ensemble(top, params, sto.RunConfig(n=n, steps=20, dt=1e-11,
                                                          record_stride=5))
    assert info.value.member == 3
    assert info.value.step == 5 and info.value.oscillator == 0


def test_ensemble_stops_at_first_diverged_record(sto):
    """The run ends at the first recording step with a non-finite state
    (integrator.py:174-177) instead of integrating NaNs to the horizon: 2e6 RK4
    steps (~10 s if run out) with a member blowing up at step 1 must return at
    once.  Members in other half-columns stop there too."""
    import time

    n, steps = 16, 2_000_000
    top = sto.Topology.decoupled(n)
    params = [sto.PhysicalParams()] * 100 + [sto.PhysicalParams(h_appl=1e300)]
    cfg = sto.RunConfig(n=n, steps=steps, dt=1e-11, record_stride=5)
    sto.integrate_ensemble(top, params[:4], sto.RunConfig(n=n, steps=10, dt=1e-11))  # warm-up
    t0 = time.perf_counter()
    with pytest.raises(sto.IntegrationDivergedError) as info:
        sto.integrate_ensemble(top, params, cfg)
    elapsed = time.perf_counter() - t0
    assert info.value.member == 100 and info.value.step == 5
    assert elapsed < 2.0, f"diverged ensemble took {elapsed:.2f} s: it did not stop early"


def test_ensemble_divergence_earliest_step_across_half_columns(sto):
    """Two members in different half-columns diverge at different recording
    steps (per-member drives blow up at different samples): the reported
    divergence is the earliest step, whichever half-column runs ahead."""
    n, batch, sps = 16, 160, 5
    top = sto.Topology(sto.CouplingMatrix.zeros(n), sto.InputWeights(np.ones((n, 1))))
    params = [sto.PhysicalParams()] * batch
    series = []
    for b in range(batch):
        u = np.zeros((40, 1))
        if b == 3:
            u[6:] = 1e300   # diverges in step 31..35 -> recording step 35
        if b == 130:
            u[2:] = 1e300   # diverges in step 11..15 -> recording step 15
        series.append(sto.InputSeries(u, sps))
    cfg = sto.RunConfig(n=n, steps=200, dt=1e-11, record_stride=5)
    with pytest.raises(sto.IntegrationDivergedError) as info:
        sto.integrate_ensemble(top, params, cfg, input_series=series)
    assert info.value.member == 130 and info.value.step == 15


@pytest.mark.parametrize("exact", [False, True])
def test_divergence_across_launches(sto, monkeypatch, exact):
    """Members split over several sequential launches (DMMA: 8 member columns
    per launch at N = 1000; exact: one member tile per launch): a member of a
    LATER launch that diverges at an EARLIER step is still the one reported."""
    if exact:
        monkeypatch.setenv("STO_EX_CT_PER_LAUNCH", "1")
    n, batch, sps = 1000, 640, 5
    w_in = np.ones((n, 1))
    top = sto.Topology(sto.CouplingMatrix.zeros(n), sto.InputWeights(w_in))
    params = [sto.PhysicalParams()] * batch
    series = []
    for b in range(batch):
        u = np.zeros((12, 1))
        if b == 3:
            u[6:] = 1e300    # launch 1: diverges in steps 31..35 -> recording step 35
        if b == 600:
            u[2:] = 1e300    # last launch: steps 11..15 -> recording step 15
        series.append(sto.InputSeries(u, sps))
    cfg = sto.RunConfig(n=n, steps=60, dt=1e-11, record_stride=5)
    with pytest.raises(sto.IntegrationDivergedError) as info:
        sto.integrate_ensemble(top, params, cfg, input_series=series, exact=exact)
    assert info.value.member == 600 and info.value.step == 15


def _rand_top(sto, n, n_in=1, seed=0):
    g = np.random.default_rng(seed)
    w = g.uniform(-1, 1, (n, n)) / np.sqrt(max(n, 3) / 3.0)
    np.fill_diagonal(w, 0.0)
    return sto.Topology(sto.CouplingMatrix(w), sto.InputWeights(g.uniform(-1, 1, (n, n_in))))


def _check_members(sto, oracle_mod, top, params, cfg, members, series=None):
    ens = sto.integrate_ensemble(top, params, cfg)
    n = cfg.n
    samples = cfg.input_series.samples if cfg.input_series is not None else np.zeros((1, top.n_in))
    sps = cfg.input_series.steps_per_sample if cfg.input_series is not None else 1
    worst = 0.0
    for b in members:
        want, _ = oracle_mod.integrate(top.coupling.entries, top.input_weights.entries,
                                       sto.kernel_scalars(params[b]), sto.initial_state(n),
                                       samples, sps, cfg.dt, cfg.steps, cfg.record_stride)
        dev = float(np.abs(ens.states[:, b] - want).max())
        worst = max(worst, dev)
        assert dev <= TOL, f"member {b}: deviation {dev:.3e}"
    return worst


@pytest.mark.parametrize("u", range(1, 8))
def test_every_tile_height(sto, oracle_mod, monkeypatch, u):
    """Force each CTA tile height TR = 8U (STO_ENS_U); n = 203 leaves a ragged last tile
    and a K tail that is not a multiple of the 32-column chunk."""
    monkeypatch.setenv("STO_ENS_U", str(u))
    n, batch, steps = 203, 70, 150
    top = _rand_top(sto, n, seed=u)
    params = _sweep(sto, batch)
    cfg = sto.RunConfig(n=n, steps=steps, dt=1e-11, record_stride=50)
    _check_members(sto, oracle_mod, top, params, cfg, [0, 33, 63, 64, 69])


@pytest.mark.parametrize("n,batch", [(1, 3), (7, 130), (8, 64), (33, 65), (1001, 4)])
def test_ragged_sizes(sto, oracle_mod, n, batch):
    top = _rand_top(sto, n, seed=n)
    params = _sweep(sto, batch)
    series = sto.InputSeries(np.random.default_rng(n).uniform(-1, 1, (20, 1)), 10)
    cfg = sto.RunConfig(n=n, steps=200, dt=1e-11, record_stride=40, input_series=series)
    members = sorted({0, batch // 2, batch - 1})
    _check_members(sto, oracle_mod, top, params, cfg, members)


def test_multichannel_input(sto, oracle_mod):
    n, n_in = 150, 3
    top = _rand_top(sto, n, n_in=n_in, seed=9)
    params = _sweep(sto, 20)
    series = sto.InputSeries(np.random.default_rng(9).uniform(-1, 1, (25, n_in)), 4)
    cfg = sto.RunConfig(n=n, steps=100, dt=1e-11, record_stride=25, input_series=series)
    _check_members(sto, oracle_mod, top, params, cfg, [0, 7, 19])


def test_several_launches(sto, oracle_mod):
    """n = 2000, B = 1024: more member columns than fit one wave of CTAs -> the host
    splits the batch into several persistent launches (member0 offsets)."""
    n, batch = 2000, 1024
    top = _rand_top(sto, n, seed=4)
    params = _sweep(sto, batch)
    cfg = sto.RunConfig(n=n, steps=20, dt=1e-11, record_stride=10)
    _check_members(sto, oracle_mod, top, params, cfg, [0, 300, 511, 512, 1023])


def test_repeat_runs_identical(sto):
    top = _rand_top(sto, 300, seed=6)
    params = _sweep(sto, 100)
    cfg = sto.RunConfig(n=300, steps=60, dt=1e-11, record_stride=20)
    a = sto.integrate_ensemble(top, params, cfg).states
    b = sto.integrate_ensemble(top, params, cfg).states
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


from hypothesis import HealthCheck, given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402


@settings(max_examples=fuzz_examples(30), deadline=None, suppress_health_check=[HealthCheck.too_slow,
                                                                 HealthCheck.function_scoped_fixture])
@given(n=st.integers(1, 260), batch=st.integers(1, 150), steps=st.integers(1, 80),
       u=st.one_of(st.none(), st.integers(1, 7)), seed=st.integers(0, 2**31 - 1))
def test_random_ensembles_within_tolerance(sto, oracle_mod, monkeypatch, n, batch, steps, u, seed):
    """Hypothesis-drawn N, B, horizon, tile height (or the host's choice) and drive:
    sampled members within the 1e-10 bar of the oracle."""
    if u is None:
        monkeypatch.delenv("STO_ENS_U", raising=False)
    else:
        monkeypatch.setenv("STO_ENS_U", str(u))
    g = np.random.default_rng(seed)
    top = _rand_top(sto, n, seed=seed)
    params = [sto.PhysicalParams(current=c) for c in g.uniform(2.0e-3, 3.0e-3, batch)]
    sps = int(g.integers(1, 5))
    series = sto.InputSeries(g.uniform(-1, 1, (-(-steps // sps), 1)), sps)
    stride = int(g.integers(1, steps + 1))
    cfg = sto.RunConfig(n=n, steps=steps, dt=1e-11, record_stride=stride, input_series=series)
    members = sorted({0, batch - 1, int(g.integers(0, batch))})
    _check_members(sto, oracle_mod, top, params, cfg, members)
