"""Bit-exact ensemble mode (integrate_ensemble(..., exact=True),
sto_ensemble_exact.cuh): every member's recorded states must equal the pinned
oracle run with that member's parameters and drive BIT FOR BIT -- at the
benched configs[3] (N = 1000, B = 512, seed-0 W) over the benched 1e4-step
horizon, and over ragged sizes, multi-channel and per-member drives, several
launches, divergence.  Oracle: oracle/sto_oracle.c, pinned to the reference's
fixtures (tests/test_oracle.py).
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import assert_bit_equal, fuzz_examples

pytestmark = pytest.mark.gpu

hypothesis = pytest.importorskip("hypothesis")
from hypothesis import HealthCheck, given, settings, strategies as st  # noqa: E402


@pytest.fixture(scope="module")
def sto():
    import paper_2312_01121_b200 as sto

    return sto


def _sweep(sto, batch):
    return [sto.PhysicalParams(current=c) for c in np.linspace(2.0e-3, 3.0e-3, batch)]


def _rand_top(sto, n, n_in=1, seed=0):
    g = np.random.default_rng(seed)
    w = g.uniform(-1, 1, (n, n)) / np.sqrt(max(n, 3) / 3.0)
    np.fill_diagonal(w, 0.0)
    return sto.Topology(sto.CouplingMatrix(w), sto.InputWeights(g.uniform(-1, 1, (n, n_in))))


def _check(sto, oracle_mod, top, params, cfg, members, series=None):
    ens = sto.integrate_ensemble(top, params, cfg, input_series=series, exact=True)
    n = cfg.n
    for b in members:
        s = series[b] if isinstance(series, list) else (series if series is not None
                                                        else cfg.input_series)
        samples = s.samples if s is not None else np.zeros((1, top.n_in))
        sps = s.steps_per_sample if s is not None else 1
        want, _ = oracle_mod.integrate(top.coupling.entries, top.input_weights.entries,
                                       sto.kernel_scalars(params[b]), sto.initial_state(n),
                                       samples, sps, cfg.dt, cfg.steps, cfg.record_stride)
        assert_bit_equal(ens.states[:, b], want, f"member {b}")
    return ens


def test_benched_config_bit_exact_at_benched_horizon(sto, oracle_mod):
    """configs[3] as benched (bench.py ens512 --exact): N = 1000, B = 512, the
    2.0-3.0 mA sweep, build_topology(1000, seed=0), 1e4 RK4 steps: sampled
    members bit-identical to the oracle at every recorded step."""
    n, batch, steps = 1000, 512, 10_000
    top = sto.build_topology(n, seed=0)
    params = _sweep(sto, batch)
    cfg = sto.RunConfig(n=n, steps=steps, dt=1e-11, record_stride=2000)
    _check(sto, oracle_mod, top, params, cfg, (0, 73, 255, 256, 438, 511))


def test_every_member_bit_exact_with_drive(sto, oracle_mod):
    n, batch, steps = 100, 70, 1000
    top = sto.build_topology(n, seed=n)
    series = sto.InputSeries(np.random.default_rng(5).uniform(-1, 1, (steps, 1)), 1)
    cfg = sto.RunConfig(n=n, steps=steps, dt=1e-11, record_stride=100, input_series=series)
    _check(sto, oracle_mod, top, _sweep(sto, batch), cfg, range(batch))


@pytest.mark.parametrize("n,batch", [(1, 3), (31, 65), (33, 64), (257, 130), (1500, 9)])
def test_ragged_sizes(sto, oracle_mod, n, batch):
    top = _rand_top(sto, n, seed=n)
    series = sto.InputSeries(np.random.default_rng(n).uniform(-1, 1, (40, 1)), 3)
    cfg = sto.RunConfig(n=n, steps=120, dt=1e-11, record_stride=40, input_series=series)
    members = sorted({0, batch // 2, batch - 1})
    _check(sto, oracle_mod, top, _sweep(sto, batch), cfg, members)


def test_multichannel_and_per_member_drives(sto, oracle_mod):
    n, batch, steps = 96, 6, 90
    top = _rand_top(sto, n, n_in=3, seed=7)
    g = np.random.default_rng(8)
    series = [sto.InputSeries(g.uniform(-1, 1, (30, 3)), 3) for _ in range(batch)]
    cfg = sto.RunConfig(n=n, steps=steps, dt=1e-11, record_stride=30)
    _check(sto, oracle_mod, top, _sweep(sto, batch), cfg, range(batch), series=series)


@pytest.mark.parametrize("u", [1, 2, 3, 4, 5, 6, 7])
def test_every_tile_height(sto, oracle_mod, monkeypatch, u):
    """Tiles of 8U oscillators x 64 members (the host picks U per size; every
    U forced here) at a ragged n with several row tiles."""
    monkeypatch.setenv("STO_EX_U", str(u))
    n, batch = 203, 70
    top = _rand_top(sto, n, seed=u)
    series = sto.InputSeries(np.random.default_rng(u).uniform(-1, 1, (30, 1)), 2)
    cfg = sto.RunConfig(n=n, steps=60, dt=1e-11, record_stride=20, input_series=series)
    _check(sto, oracle_mod, top, _sweep(sto, batch), cfg, (0, 37, 64, 69))


def test_many_tiles_per_cta(sto, oracle_mod, monkeypatch):
    """More tiles than SMs: every CTA walks several tiles per stage (here 8-row
    tiles, N = 1000, B = 640 -> 1250 tiles, ~9 per CTA), including the per-
    column counters of tiles that share a CTA."""
    monkeypatch.setenv("STO_EX_U", "1")
    n, batch, steps = 1000, 640, 30
    top = _rand_top(sto, n, seed=41)
    series = sto.InputSeries(np.random.default_rng(42).uniform(-1, 1, (steps, 1)), 1)
    cfg = sto.RunConfig(n=n, steps=steps, dt=1e-11, record_stride=10, input_series=series)
    _check(sto, oracle_mod, top, _sweep(sto, batch), cfg, (0, 63, 64, 333, 639))


def test_many_tiles_per_cta_divergence(sto, monkeypatch):
    """Record-step stop with several tiles per CTA: only the diverging member's
    column stops early, the others run on; the earliest (step, member) wins."""
    monkeypatch.setenv("STO_EX_U", "1")
    n, batch = 64, 2500  # 8 row tiles x 40 member tiles = 320 tiles > 148 CTAs
    top = sto.Topology(sto.CouplingMatrix.zeros(n), sto.InputWeights(np.ones((n, 1))))
    params = [sto.PhysicalParams()] * batch
    series = []
    for b in range(batch):
        u = np.zeros((20, 1))
        if b == 2400:
            u[3:] = 1e300   # diverges in steps 16..20 -> recording step 20
        if b == 7:
            u[7:] = 1e300   # later: steps 36..40 -> recording step 40
        series.append(sto.InputSeries(u, 5))
    cfg = sto.RunConfig(n=n, steps=100, dt=1e-11, record_stride=5)
    with pytest.raises(sto.IntegrationDivergedError) as info:
        sto.integrate_ensemble(top, params, cfg, input_series=series, exact=True)
    assert info.value.member == 2400 and info.value.step == 20


def test_several_launches(sto, oracle_mod, monkeypatch):
    monkeypatch.setenv("STO_EX_CT_PER_LAUNCH", "1")
    n, batch = 64, 150
    top = _rand_top(sto, n, seed=11)
    cfg = sto.RunConfig(n=n, steps=60, dt=1e-11, record_stride=20)
    _check(sto, oracle_mod, top, _sweep(sto, batch), cfg, (0, 63, 64, 127, 128, 149))


def test_custom_initial_states_bit_exact(sto, oracle_mod):
    """integrate_ensemble(m0=...) with one random unit-norm start per member:
    each member equals the oracle run from that start (the f4 extension of
    integrate(m0=) carried to ensembles)."""
    n, batch, steps = 70, 5, 80
    top = _rand_top(sto, n, seed=21)
    g = np.random.default_rng(22)
    m0 = g.normal(size=(batch, n, 3))
    m0 /= np.linalg.norm(m0, axis=2, keepdims=True)
    params = _sweep(sto, batch)
    cfg = sto.RunConfig(n=n, steps=steps, dt=1e-11, record_stride=20)
    ens = sto.integrate_ensemble(top, params, cfg, exact=True, m0=m0)
    for b in range(batch):
        want, _ = oracle_mod.integrate(top.coupling.entries, top.input_weights.entries,
                                       sto.kernel_scalars(params[b]), m0[b], np.zeros((1, 1)), 1,
                                       1e-11, steps, 20)
        assert_bit_equal(ens.states[:, b], want, f"member {b}")
    with pytest.raises(sto.ParameterError):
        sto.integrate_ensemble(top, params, cfg, m0=m0[:, :10])


def test_matches_dmma_path_within_tolerance(sto):
    n, batch = 200, 64
    top = sto.build_topology(n, seed=4)
    cfg = sto.RunConfig(n=n, steps=500, dt=1e-11, record_stride=100)
    a = sto.integrate_ensemble(top, _sweep(sto, batch), cfg, exact=True)
    b = sto.integrate_ensemble(top, _sweep(sto, batch), cfg)
    assert float(np.abs(a.states - b.states).max()) <= 1e-10


def test_exact_divergence_reports_first_member_and_stops(sto):
    import time

    n, steps = 16, 2_000_000
    top = sto.Topology.decoupled(n)
    params = [sto.PhysicalParams()] * 100 + [sto.PhysicalParams(h_appl=1e300)]
    cfg = sto.RunConfig(n=n, steps=steps, dt=1e-11, record_stride=5)
    sto.integrate_ensemble(top, params[:4], sto.RunConfig(n=n, steps=10, dt=1e-11), exact=True)
    t0 = time.perf_counter()
    with pytest.raises(sto.IntegrationDivergedError) as info:
        sto.integrate_ensemble(top, params, cfg, exact=True)
    assert info.value.member == 100 and info.value.step == 5 and info.value.oscillator == 0
    assert time.perf_counter() - t0 < 2.0


@settings(max_examples=fuzz_examples(25), deadline=None, suppress_health_check=list(HealthCheck))
@given(n=st.integers(1, 300), batch=st.integers(1, 400), steps=st.integers(1, 60),
       stride=st.integers(1, 25), sps=st.integers(1, 7), u=st.integers(0, 7),
       seed=st.integers(0, 2**31 - 1))
def test_random_exact_ensembles(sto, oracle_mod, n, batch, steps, stride, sps, u, seed):
    """Random sizes, drives, member parameters and tile heights (u = 0: the
    host's choice; small u with large B gives several tiles per CTA)."""
    import os

    g = np.random.default_rng(seed)
    top = _rand_top(sto, n, seed=seed)
    params = [sto.PhysicalParams(current=float(c), h_appl=float(h))
              for c, h in zip(g.uniform(1e-3, 4e-3, batch), g.uniform(0, 500, batch))]
    series = sto.InputSeries(g.uniform(-1, 1, ((steps + sps - 1) // sps, 1)), sps)
    cfg = sto.RunConfig(n=n, steps=steps, dt=1e-11, record_stride=stride, input_series=series)
    old = os.environ.get("STO_EX_U")
    if u:
        os.environ["STO_EX_U"] = str(u)
    try:
        _check(sto, oracle_mod, top, params, cfg, sorted({0, batch - 1, int(g.integers(batch))}))
    finally:
        if old is None:
            os.environ.pop("STO_EX_U", None)
        else:
            os.environ["STO_EX_U"] = old
