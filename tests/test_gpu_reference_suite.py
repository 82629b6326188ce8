"""The reference's own integrator / acceptance checks, re-pointed at the B200 path.

Modelled on spinosc's tests: test_integrator.py (rigid rotation :127-144,
norm conservation :146-150, single-step drift :154-165, recording grid
:99-120, validation :200-212) and test_acceptance.py (A1 norm drift, A4
integrator order :130-150, A6 oscillation onset :177-201, A9 decoupled
independence :243-261). Every run here goes through the public
`integrate()` and the persistent kernels.
"""

from __future__ import annotations

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sto():
    import paper_2312_01121_b200 as sto

    return sto


def _precession_params(sto):
    # alpha = 0, I = 0, H_K = 4 pi M: the field is h_appl e_z, closed-form rotation
    return sto.PhysicalParams(alpha=0.0, current=0.0, h_k=4.0 * math.pi * 1448.3)


def test_rigid_rotation_closed_form(sto):
    params = _precession_params(sto)
    traj = sto.integrate(sto.Topology.decoupled(1), params,
                         sto.RunConfig(n=1, steps=400, dt=1e-12, record_stride=40))
    omega = params.gamma * params.h_appl
    m0 = sto.initial_state(1)[0]
    for i, t in enumerate(traj.times):
        c, s = math.cos(omega * t), math.sin(omega * t)
        want = np.array([m0[0] * c - m0[1] * s, m0[0] * s + m0[1] * c, m0[2]])
        assert np.abs(traj.states[i, 0] - want).max() <= 1e-12


def test_norm_conserved_without_torque(sto):
    traj = sto.integrate(sto.Topology.decoupled(1), _precession_params(sto),
                         sto.RunConfig(n=1, steps=400, dt=1e-12))
    assert traj.max_norm_drift <= 1e-13


def test_single_step_drift_window(sto):
    p = sto.PhysicalParams()
    coarse = sto.integrate(sto.Topology.decoupled(1), p, sto.RunConfig(n=1, steps=1, dt=1e-11))
    assert 1e-10 <= coarse.max_norm_drift <= 1e-9
    fine = sto.integrate(sto.Topology.decoupled(1), p, sto.RunConfig(n=1, steps=2, dt=5e-12))
    assert fine.max_norm_drift < coarse.max_norm_drift / 16.0


def test_a1_norm_drift_n10(sto):
    traj = sto.run(sto.RunConfig(n=10, steps=10_000, dt=1e-11, seed=0))
    # the reference documents ~2e-6 per 1e4 steps at dt=1e-11 (README known deviations);
    # the GPU must reproduce exactly the same drift as its bit-exact oracle, i.e. the same band
    assert 1e-6 <= traj.max_norm_drift <= 5e-6


def test_a4_integrator_order(sto):
    top = sto.build_topology(1, seed=0)
    p = sto.PhysicalParams()

    def final_at(refine):
        cfg = sto.RunConfig(n=1, steps=1000 * refine, dt=2e-12 / refine,
                            record_stride=1000 * refine)
        return sto.integrate(top, p, cfg).final_state

    ref = final_at(8)
    dts = np.array([2e-12, 1e-12, 5e-13])
    errs = np.array([np.abs(final_at(r) - ref).max() for r in (1, 2, 4)])
    slope = float(np.polyfit(np.log(dts), np.log(errs), 1)[0])
    assert 3.7 <= slope <= 4.3


def test_a6_oscillation_sign_changes(sto):
    traj = sto.integrate(sto.build_topology(1, seed=0), sto.PhysicalParams(),
                         sto.RunConfig(n=1, steps=10_000, dt=1e-11))
    mx = traj.states[:, 0, 0]
    signs = np.sign(mx[mx != 0.0])
    assert int(np.count_nonzero(np.diff(signs))) >= 50


def test_recording_grid_with_remainder(sto):
    top = sto.build_topology(5, seed=1)
    traj = sto.integrate(top, sto.PhysicalParams(),
                         sto.RunConfig(n=5, steps=10, dt=1e-11, record_stride=3))
    assert list(np.round(traj.times / 1e-11).astype(int)) == [0, 3, 6, 9, 10]
    assert traj.states.shape == (5, 5, 3)


def test_validation_errors_reach_the_user(sto):
    with pytest.raises(sto.ParameterError):
        sto.integrate(sto.Topology.decoupled(3), sto.PhysicalParams(),
                      sto.RunConfig(n=3, steps=7, dt=1e-11,
                                    input_series=sto.InputSeries(np.ones((3, 1)), 1)))


def test_backend_reports_plan(sto):
    be = sto.create_backend("gpu", sto.build_topology(1000, seed=0), sto.PhysicalParams())
    info = be.plan_info
    assert info["kernel_name"] == "reg" and info["grid"] >= 64
    be10k = sto.create_backend("gpu", sto.Topology.decoupled(10_000), sto.PhysicalParams())
    assert be10k.plan_info["kernel_name"] == "stream"
