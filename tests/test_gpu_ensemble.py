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

pytestmark = pytest.mark.gpu

TOL = 1e-10


@pytest.fixture(scope="module")
def sto():
    import paper_2312_01121_b200 as sto

    return sto


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
