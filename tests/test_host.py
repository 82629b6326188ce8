"""Host-side mirror of the reference API (no GPU needed).

Parameters, topology construction (pinned bit-exactly against W matrices the
reference built), drive series, run configuration, recording grid, the
backend registry and the stage-wise path for derivative-only plugins --
modelled on the reference's own test_params / test_topology / test_model /
test_integrator / test_backends suites.
"""

from __future__ import annotations

import math

import numpy as np
import pytest

import paper_2312_01121_b200 as sto
from paper_2312_01121_b200 import (BackendUnavailableError, InputSeries,
                                   IntegrationDivergedError, ParameterError, PhysicalParams,
                                   RunConfig, Topology, TrajectoryMismatchError,
                                   compare_trajectories, integrate)
from paper_2312_01121_b200.integrator import RK4Scratch, _recorded_steps, rk4_step
from paper_2312_01121_b200.topology import (CouplingMatrix, InputWeights, RngStream,
                                            build_topology, initial_state, spectral_radius)

from conftest import assert_bit_equal, load_golden


# ---------------------------------------------------------------- params ----
def test_derived_constants_match_reference_freeze():
    d = sto.derive(PhysicalParams())
    # frozen in the reference's test_params.py:15-19
    assert d.c_prec == pytest.approx(17639559.011024725, rel=1e-15)
    assert d.c_damp == pytest.approx(88197.79505512363, rel=1e-15)
    assert d.h_aniso == pytest.approx(416.12543922361147, rel=1e-15)
    assert d.h_s_prefactor == pytest.approx(134.86812645902467, rel=1e-15)
    assert sto.small_angle_frequency(PhysicalParams()) == pytest.approx(1.729767978589695e9,
                                                                        rel=1e-12)


def test_kernel_scalars_bit_equal_reference_pack():
    # consts stored by make_golden.py come from the reference's _scalar_pack
    z = load_golden("deriv.npz")
    assert_bit_equal(np.array(sto.kernel_scalars(PhysicalParams())), z["consts"])
    d = load_golden("traj_n160_params.npz")
    p = PhysicalParams(alpha=0.01, current=3.0e-3, a_cp=2.0, a_in=0.5)
    assert_bit_equal(np.array(sto.kernel_scalars(p)), d["consts"])


@pytest.mark.parametrize("kwargs", [{"gamma": 0.0}, {"alpha": -1e-3}, {"lambda_stt": 1.0},
                                    {"h_appl": float("nan")}, {"current": float("inf")},
                                    {"p_vec": (0.0, 0.0, 0.0)}, {"volume": -1.0}])
def test_params_validation(kwargs):
    with pytest.raises(ParameterError):
        PhysicalParams(**kwargs)


# -------------------------------------------------------------- topology ----
@pytest.mark.parametrize("n,n_in,seed", [(1, 1, 0), (2, 1, 1), (3, 1, 3), (6, 2, 5), (7, 1, 11),
                                         (13, 1, 7), (33, 3, 33), (100, 1, 0), (160, 1, 3)])
def test_build_topology_bit_equal_reference(n, n_in, seed):
    ref = load_golden(f"topo_n{n}_in{n_in}_s{seed}.npz")
    top = build_topology(n, n_in=n_in, seed=seed)
    assert_bit_equal(top.coupling.entries, ref["w"], "W")
    assert_bit_equal(top.input_weights.entries, ref["w_in"], "W_in")


def test_rng_frozen_draws():
    # reference test_topology.py:36-42
    want = np.array([0.2739233746429086, -0.4604265724722594, -0.9180529521276106,
                     -0.9669447289429418])
    assert np.array_equal(RngStream(0).uniform_pm1(4), want)


def test_spectral_radius_cases():
    assert spectral_radius(np.array([[0.0, 0.7], [-0.3, 0.0]])) == pytest.approx(math.sqrt(0.21))
    assert spectral_radius(np.zeros((6, 6))) == 0.0
    shift = np.zeros((8, 8))
    shift[np.arange(7), np.arange(1, 8)] = 1.0
    assert spectral_radius(shift) == 0.0
    g = np.random.default_rng(4)
    w = g.uniform(-1, 1, (40, 40))
    assert spectral_radius(w) == pytest.approx(np.abs(np.linalg.eigvals(w)).max(), rel=1e-8)


def test_containers_validate():
    with pytest.raises(ParameterError):
        CouplingMatrix(entries=np.ones((2, 2)))
    with pytest.raises(ParameterError):
        InputWeights(entries=np.full((2, 1), 1.5))
    with pytest.raises(ParameterError):
        Topology(CouplingMatrix.zeros(3), InputWeights.zeros(4))
    t = Topology.decoupled(5, n_in=2)
    assert (t.n, t.n_in) == (5, 2)


def test_initial_state_unit_norm():
    m = initial_state(4)
    assert m.shape == (4, 3)
    assert np.allclose(np.linalg.norm(m, axis=1), 1.0, atol=1e-15)


# ------------------------------------------------------------ drive/config ----
def test_input_series_hold_and_bounds():
    s = InputSeries(samples=np.array([[1.0], [2.0], [3.0]]), steps_per_sample=4)
    assert [s.sample_for_step(i)[0] for i in range(12)] == [1.0] * 4 + [2.0] * 4 + [3.0] * 4
    s.check_steps(9)
    s.check_steps(12)
    for bad in (8, 13):
        with pytest.raises(ParameterError):
            s.check_steps(bad)
    with pytest.raises(ParameterError):
        InputSeries(samples=np.array([[np.inf]]))


@pytest.mark.parametrize("kwargs", [{"n": 0, "steps": 1, "dt": 1e-11},
                                    {"n": 1, "steps": 0, "dt": 1e-11},
                                    {"n": 1, "steps": 1, "dt": 0.0},
                                    {"n": 1, "steps": 1, "dt": float("inf")},
                                    {"n": 1, "steps": 1, "dt": 1e-11, "record_stride": 0},
                                    {"n": 1, "steps": 1, "dt": 1e-11, "workers": 0}])
def test_run_config_rejects(kwargs):
    with pytest.raises(ParameterError):
        RunConfig(**kwargs)


def test_recording_grid():
    assert list(_recorded_steps(5, 1)) == [0, 1, 2, 3, 4, 5]
    assert list(_recorded_steps(10, 3)) == [0, 3, 6, 9, 10]
    assert list(_recorded_steps(5, 100)) == [0, 5]


# -------------------------------------------------------------- registry ----
def test_registry_lists_gpu_backend():
    ids = [d.backend_id for d in sto.list_backends()]
    assert ids == ["gpu"]


def test_unknown_backend_raises_listing_alternatives(params):
    with pytest.raises(BackendUnavailableError) as info:
        sto.create_backend("quantum", Topology.decoupled(1), params)
    assert info.value.requested == "quantum"


def test_register_replace_unregister(params):
    class Zero:
        def derivative(self, m, u, out):
            out.fill(0.0)
            return out

    sto.register_backend("stub", kind="test double", requires="nothing", probe=lambda: True,
                         factory=lambda top, par, **kw: Zero())
    try:
        assert "stub" in sto.available_backend_ids()
        traj = integrate(Topology.decoupled(3), params,
                         RunConfig(n=3, steps=20, dt=1e-11, backend="stub"))
        assert np.array_equal(traj.states[-1], traj.states[0])
    finally:
        sto.unregister_backend("stub")
    assert "stub" not in sto.available_backend_ids()


def test_probe_that_raises_counts_as_unavailable(params):
    def boom():
        raise RuntimeError("probe exploded")

    sto.register_backend("flaky", kind="t", requires="t", probe=boom, factory=lambda *a, **k: 0)
    try:
        assert "flaky" not in sto.available_backend_ids()
        with pytest.raises(BackendUnavailableError):
            sto.create_backend("flaky", Topology.decoupled(1), params)
    finally:
        sto.unregister_backend("flaky")


# --------------------------------------------- derivative-only plugin path ----
class _Stub:
    def __init__(self, fn):
        self.fn, self.calls, self.seen_u = fn, 0, []

    def derivative(self, m, u, out):
        self.calls += 1
        self.seen_u.append(float(u[0]))
        self.fn(m, u, out)
        return out


def test_plugin_zero_derivative_fixed_point(params):
    stub = _Stub(lambda m, u, out: out.fill(0.0))
    traj = integrate(Topology.decoupled(3), params, RunConfig(n=3, steps=50, dt=1e-11),
                     backend=stub)
    assert np.array_equal(traj.states[-1], traj.states[0])
    assert stub.calls == 200 and traj.max_norm_drift == 0.0


def test_plugin_zoh_held_across_stages(params):
    series = InputSeries(samples=np.array([[10.0], [20.0]]), steps_per_sample=2)
    stub = _Stub(lambda m, u, out: out.fill(0.0))
    integrate(Topology.decoupled(1), params,
              RunConfig(n=1, steps=4, dt=1e-11, input_series=series), backend=stub)
    assert stub.seen_u == [10.0] * 8 + [20.0] * 8


def test_rk4_step_is_degree4_taylor():
    m = np.full((2, 3), 1.0)
    rk4_step(lambda s, u, out: np.multiply(s, -2.0, out=out), m, np.zeros(1), 0.125,
             RK4Scratch(2))
    x = -0.25
    assert np.abs(m - (1 + x + x**2 / 2 + x**3 / 6 + x**4 / 24)).max() <= 1e-16


def test_plugin_divergence_location(params):
    def poison(m, u, out):
        out.fill(0.0)
        out[2, 0] = np.inf

    with pytest.raises(IntegrationDivergedError) as info:
        integrate(Topology.decoupled(4), params, RunConfig(n=4, steps=5, dt=1e-11),
                  backend=_Stub(poison))
    assert (info.value.oscillator, info.value.step) == (2, 1)


def test_validation_errors(params):
    with pytest.raises(ParameterError):
        integrate(Topology.decoupled(3), params, RunConfig(n=4, steps=1, dt=1e-11))
    with pytest.raises(ParameterError):
        integrate(Topology.decoupled(3), params,
                  RunConfig(n=3, steps=1, dt=1e-11, input_series=InputSeries.zeros(2)))
    with pytest.raises(ParameterError):
        integrate(Topology.decoupled(1), params,
                  RunConfig(n=1, steps=7, dt=1e-11,
                            input_series=InputSeries(np.ones((3, 1)), 1)))


def test_compare_trajectories_grid_checks(params):
    stub = _Stub(lambda m, u, out: out.fill(0.0))
    a = integrate(Topology.decoupled(2), params, RunConfig(n=2, steps=10, dt=1e-11), backend=stub)
    b = integrate(Topology.decoupled(2), params, RunConfig(n=2, steps=11, dt=1e-11), backend=stub)
    c = integrate(Topology.decoupled(2), params, RunConfig(n=2, steps=10, dt=2e-11), backend=stub)
    assert compare_trajectories(a, a) == 0.0
    for other in (b, c):
        with pytest.raises(TrajectoryMismatchError):
            compare_trajectories(a, other)


def test_trajectory_csv_round_trip(tmp_path, params):
    stub = _Stub(lambda m, u, out: np.multiply(m, -1e9, out=out))
    traj = integrate(Topology.decoupled(2), params, RunConfig(n=2, steps=3, dt=1e-11),
                     backend=stub)
    path = tmp_path / "t.csv"
    sto.write_trajectory_csv(path, traj)
    lines = path.read_text().splitlines()
    assert lines[0] == "t,k,mx,my,mz" and len(lines) == 1 + traj.n_recorded * 2
    t, k, mx, my, mz = lines[-1].split(",")
    assert float(t) == traj.times[-1] and int(k) == 1
    assert (float(mx), float(my), float(mz)) == tuple(traj.states[-1, 1])


def _pcg_restated(state: int, inc: int, count: int, offset: int = 0) -> np.ndarray:
    """Pure-Python PCG-XSL-RR 128/64 with LCG jump-ahead -- the formulas the device
    kernel (csrc/sto_build.cuh) implements -- mapped to 2u - 1."""
    mask = (1 << 128) - 1
    mult = 0x2360ED051FC65DA44385DF649FCCF645
    # jump `offset` steps
    acc_m, acc_p, cur_m, cur_p, d = 1, 0, mult, inc, offset
    while d:
        if d & 1:
            acc_m, acc_p = (acc_m * cur_m) & mask, (acc_p * cur_m + cur_p) & mask
        cur_p, cur_m, d = ((cur_m + 1) * cur_p) & mask, (cur_m * cur_m) & mask, d >> 1
    state = (acc_m * state + acc_p) & mask
    out = np.empty(count)
    for i in range(count):
        state = (state * mult + inc) & mask
        x = ((state >> 64) ^ state) & ((1 << 64) - 1)
        rot = state >> 122
        x = ((x >> rot) | (x << ((64 - rot) & 63))) & ((1 << 64) - 1)
        out[i] = 2.0 * ((x >> 11) * 2.0 ** -53) - 1.0
    return out


@pytest.mark.parametrize("seed", [0, 5, 2**33 + 1])
def test_pcg64_restatement_matches_numpy(seed):
    """Pins the device PCG64 formulas (step-then-output, XSL-RR, jump-ahead) on the
    CPU against numpy's Generator(PCG64(seed)) -- the reference's RngStream."""
    from paper_2312_01121_b200 import RngStream, _native

    hi, lo, ihi, ilo = _native.pcg64_words(seed)
    state, inc = (hi << 64) | lo, (ihi << 64) | ilo
    rs = RngStream(seed)
    assert np.array_equal(_pcg_restated(state, inc, 20), rs.uniform_pm1(20))
    rs.uniform_pm1(977)
    assert np.array_equal(_pcg_restated(state, inc, 5, offset=997), rs.uniform_pm1(5))


def _reference_csv_text(times, states) -> str:
    """The reference's write_trajectory_csv loop (integrator.py:217-225), restated."""
    lines = ["t,k,mx,my,mz\n"]
    for i in range(states.shape[0]):
        t = times[i]
        for k in range(states.shape[1]):
            mx, my, mz = states[i, k]
            lines.append(f"{t:.17g},{k},{mx:.17g},{my:.17g},{mz:.17g}\n")
    return "".join(lines)


@pytest.mark.parametrize("threads", [1, 3, 0])
def test_native_csv_writer_is_byte_identical(tmp_path, threads):
    from paper_2312_01121_b200 import _native

    g = np.random.default_rng(11)
    R, n = 7, 9000  # > one 16384-row block per thread
    states = g.standard_normal((R, n, 3)) * 10.0 ** g.integers(-320, 300, (R, n, 3))
    special = [0.0, -0.0, 1.0, -1.0, 1e-4, 9.9999999999999991e-05, 1e16, 1e17, 123456789012345678.0,
               5e-324, -2.2250738585072014e-308, 1.7976931348623157e308, 0.1, 1 / 3, np.inf,
               -np.inf, np.nan, -np.nan]
    flat = states.reshape(-1)
    flat[:len(special)] = special
    times = np.arange(R) * 1e-11 * 137
    path = tmp_path / "traj.csv"
    _native.write_trajectory_csv(path, times, states, threads=threads)
    assert path.read_text() == _reference_csv_text(times, states)


def test_write_trajectory_csv_public_api(tmp_path):
    states = np.random.default_rng(2).uniform(-1, 1, (3, 5, 3))
    traj = sto.Trajectory(times=np.array([0.0, 1e-10, 2e-10]), states=states, max_norm_drift=0.0,
                          config=sto.RunConfig(n=5, steps=20, dt=1e-11), elapsed_seconds=0.0)
    sto.write_trajectory_csv(tmp_path / "a.csv", traj)
    assert (tmp_path / "a.csv").read_text() == _reference_csv_text(traj.times, states)


class _OracleDerivative:
    """Derivative-only test double (the pinned C oracle): steps through the
    stagewise path of integrate()."""

    def __init__(self, top, params):
        from oracle import oracle

        import paper_2312_01121_b200 as sto

        self._o, self._top = oracle, top
        self._c = sto.kernel_scalars(params)

    def derivative(self, m, u, out):
        out[...] = self._o.derivative(self._top.coupling.entries, self._top.input_weights.entries,
                                      self._c, m, u)
        return out


@pytest.mark.parametrize("split,sps,stride", [(60, 3, 20), (61, 3, 61), (45, 1, 15)])
def test_resume_continues_bit_exact(params, oracle_mod, split, sps, stride):
    """f4: run(a + b) == run(a) + resume(b), bit for bit -- also when the split
    falls inside a held drive sample (61 % 3 != 0); and both equal the oracle."""
    import paper_2312_01121_b200 as sto

    n, total = 24, 120
    top = sto.build_topology(n, seed=9)
    g = np.random.default_rng(split)
    full = sto.InputSeries(g.uniform(-1, 1, (-(-total // sps), 1)), sps)
    head = sto.InputSeries(full.samples[:-(-split // sps)], sps)
    be = _OracleDerivative(top, params)
    whole = sto.integrate(top, params, sto.RunConfig(n=n, steps=total, dt=1e-11,
                                                     record_stride=stride, input_series=full),
                          backend=be)
    first = sto.integrate(top, params, sto.RunConfig(n=n, steps=split, dt=1e-11,
                                                     record_stride=stride, input_series=head),
                          backend=be)
    rest = sto.resume(first, top, params, total - split, backend=be, input_series=full)
    assert rest.step_offset == split
    got = np.concatenate([first.states, rest.states[1:]])
    times = np.concatenate([first.times, rest.times[1:]])
    assert np.array_equal(times, whole.times)
    assert np.array_equal(got.view(np.uint64), whole.states.view(np.uint64))
    want, _ = oracle_mod.integrate(top.coupling.entries, top.input_weights.entries,
                                   sto.kernel_scalars(params), sto.initial_state(n), full.samples,
                                   sps, 1e-11, total, stride)
    assert np.array_equal(whole.states.view(np.uint64), want.view(np.uint64))


def test_integrate_custom_m0_and_checks(params):
    import paper_2312_01121_b200 as sto

    n = 5
    top = sto.build_topology(n, seed=2)
    be = _OracleDerivative(top, params)
    m0 = np.random.default_rng(0).standard_normal((n, 3))
    m0 /= np.linalg.norm(m0, axis=1, keepdims=True)
    keep = m0.copy()
    traj = sto.integrate(top, params, sto.RunConfig(n=n, steps=10, dt=1e-11), backend=be, m0=m0)
    assert np.array_equal(traj.states[0], keep) and np.array_equal(m0, keep)  # m0 untouched
    with pytest.raises(sto.ParameterError):
        sto.integrate(top, params, sto.RunConfig(n=n, steps=10, dt=1e-11), backend=be,
                      m0=np.zeros((n + 1, 3)))
    with pytest.raises(sto.ParameterError):
        sto.integrate(top, params, sto.RunConfig(n=n, steps=10, dt=1e-11), backend=be,
                      step_offset=-1)


def test_resume_divergence_reports_global_step(params):
    import paper_2312_01121_b200 as sto

    def poison(m, u, out):
        out[...] = 0.0
        if u[0] > 0.5:
            out[2, 0] = np.inf

    top = sto.Topology.decoupled(4)
    drive = np.zeros((40, 1))
    drive[25:] = 1.0
    series = sto.InputSeries(drive, 1)
    first = sto.integrate(top, params, sto.RunConfig(
        n=4, steps=20, dt=1e-11, record_stride=5, input_series=sto.InputSeries(drive[:20], 1)),
        backend=_Stub(poison))
    with pytest.raises(sto.IntegrationDivergedError) as info:
        sto.resume(first, top, params, 20, backend=_Stub(poison), input_series=series)
    assert (info.value.oscillator, info.value.step) == (2, 30)


def test_numpy_norm_order_pinned():
    """Trajectory.max_norm_drift is np.linalg.norm(states, axis=-1) (ref
    integrator.py:184-185); the device version (sto_norm_drift) evaluates
    sqrt((x*x + y*y) + z*z) with every operation rounded -- numpy's order for a
    contiguous 3-element reduction.  Pin it here so a numpy change shows up."""
    g = np.random.default_rng(0)
    v = g.uniform(-1, 1, (200_000, 3)) * np.exp2(g.integers(-30, 30, (200_000, 1)))
    want = np.linalg.norm(v, axis=-1)
    got = np.sqrt((v[:, 0] * v[:, 0] + v[:, 1] * v[:, 1]) + v[:, 2] * v[:, 2])
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_integrate_ensemble_argument_checks_before_any_device_work():
    """integrate_ensemble validates its arguments (ref-style ParameterError)
    before a backend exists, so they hold on a host without a GPU."""
    import pytest

    import paper_2312_01121_b200 as sto
    from paper_2312_01121_b200.errors import ParameterError

    top = sto.Topology.decoupled(8)
    cfg = sto.RunConfig(n=8, steps=10, dt=1e-11)
    params = [sto.PhysicalParams()] * 3
    with pytest.raises(ParameterError):
        sto.integrate_ensemble(top, [], cfg)
    with pytest.raises(ParameterError):
        sto.integrate_ensemble(sto.Topology.decoupled(9), params, cfg)
    with pytest.raises(ParameterError):
        sto.integrate_ensemble(top, params, cfg, m0=np.zeros((2, 8, 3)))
    with pytest.raises(ParameterError):
        sto.integrate_ensemble(top, params, cfg,
                               input_series=[sto.InputSeries.zeros(1)] * 2)
