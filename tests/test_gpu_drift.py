"""Trajectory.max_norm_drift on the device (sto_norm_drift) against the
reference's host expression np.abs(np.linalg.norm(states, axis=-1) - 1).max()
(integrator.py:184-185): bit-equal, per trajectory and per ensemble member."""

from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _host(states, axis):
    return np.abs(np.linalg.norm(states, axis=axis) - 1.0)


def test_drift_kernel_matches_numpy():
    from paper_2312_01121_b200 import _native

    g = np.random.default_rng(1)
    for shape, members in (((7, 1, 1, 3), 1), ((101, 1, 333, 3), 1), ((5, 70, 65, 3), 70)):
        v = g.normal(size=shape)
        v /= np.linalg.norm(v, axis=-1, keepdims=True)
        v *= 1.0 + g.normal(scale=1e-7, size=shape[:-1] + (1,))
        got = _native.norm_drift(torch.from_numpy(v).cuda(), members=members).cpu().numpy()
        want = _host(v, -1).max(axis=(0, 2))
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), (shape, got, want)


def test_trajectory_drift_bit_equal_to_host_expression():
    import paper_2312_01121_b200 as sto

    n, steps = 100, 400
    top = sto.build_topology(n, seed=5)
    series = sto.InputSeries(np.random.default_rng(2).uniform(-1, 1, (steps, 1)), 1)
    tr = sto.integrate(top, sto.PhysicalParams(), sto.RunConfig(n=n, steps=steps, dt=1e-11,
                                                               record_stride=1, input_series=series))
    want = float(_host(tr.states, 2).max())
    assert np.float64(tr.max_norm_drift).view(np.uint64) == np.float64(want).view(np.uint64)
    ens = sto.integrate_ensemble(top, [sto.PhysicalParams(current=c) for c in (2e-3, 3e-3)],
                                 sto.RunConfig(n=n, steps=50, dt=1e-11, record_stride=5))
    want = _host(ens.states, 3).max(axis=(0, 2))
    assert np.array_equal(ens.max_norm_drift.view(np.uint64), want.view(np.uint64))
