"""The B200 backend inside the reference package's own registry, integrator and CLI
(paper_2312_01121_b200/spinosc_plugin.py).

CPU: registration replaces spinosc's "gpu" entry, its probe never raises and is
false without a GPU, and the whole-run hook leaves every other backend on the
reference's untouched loop (bit-identical trajectories).
GPU: `spinosc validate` passes the B200 backend against the numpy reference
(deviation 0.0), `spinosc.integrate(..., backend="gpu")` runs in one launch and
matches the reference's `fused` backend bit for bit, divergence surfaces as the
reference's IntegrationDivergedError, and `spinosc bench` reports its speedup.
"""

from __future__ import annotations

import numpy as np
import pytest


@pytest.fixture(scope="module")
def plugged(spinosc_ref):
    from paper_2312_01121_b200 import spinosc_plugin

    spinosc_plugin.register()
    spinosc_plugin.register()  # idempotent
    return spinosc_ref


def test_registered_under_reference_id(plugged):
    desc = {d.backend_id: d for d in plugged.list_backends()}
    assert desc["gpu"].kind.startswith("B200")
    import spinosc.integrator as integ

    assert getattr(integ.integrate, "__wrapped__", None) is not None
    import spinosc.cli as cli

    assert cli.integrate is integ.integrate


def test_probe_never_raises(plugged):
    from paper_2312_01121_b200 import spinosc_plugin

    assert spinosc_plugin._probe() in (True, False)


def test_hook_keeps_reference_loop_for_cpu_backends(plugged):
    sp = plugged
    top = sp.build_topology(12, seed=3)
    cfg = sp.RunConfig(n=12, steps=40, dt=1e-11, record_stride=10, backend="reference")
    import spinosc.integrator as integ

    a = integ.integrate(top, sp.PhysicalParams(), cfg)
    b = integ.integrate.__wrapped__(top, sp.PhysicalParams(), cfg)
    assert np.array_equal(a.states, b.states) and np.array_equal(a.times, b.times)


@pytest.mark.gpu
def test_reference_validate_passes_b200(plugged, capsys):
    import spinosc.cli as cli

    rc = cli.main(["validate", "--n", "100", "--steps", "1000", "--record-stride", "100"])
    out = capsys.readouterr().out
    assert rc == 0, out
    line = next(l for l in out.splitlines() if "vs gpu" in l)
    assert "max deviation 0.000e+00" in line and "PASS" in line


@pytest.mark.gpu
def test_reference_integrate_whole_run_bit_exact(plugged):
    sp = plugged
    top = sp.build_topology(300, seed=1)
    series = sp.InputSeries(np.random.default_rng(2).uniform(-1, 1, (100, 1)), 5)
    cfg = sp.RunConfig(n=300, steps=500, dt=1e-11, record_stride=50, input_series=series,
                       backend="gpu")
    g = sp.integrate(top, sp.PhysicalParams(), cfg)
    f = sp.integrate(top, sp.PhysicalParams(), cfg.with_overrides(backend="fused"))
    assert type(g) is type(f)
    assert np.array_equal(g.states.view(np.uint64), f.states.view(np.uint64))
    assert np.array_equal(g.times, f.times) and g.max_norm_drift == f.max_norm_drift


@pytest.mark.gpu
def test_reference_divergence_error(plugged):
    sp = plugged
    params = sp.PhysicalParams().with_overrides(h_appl=1e300)
    cfg = sp.RunConfig(n=4, steps=30, dt=1e-11, record_stride=10, backend="gpu")
    with pytest.raises(sp.IntegrationDivergedError) as info:
        sp.integrate(sp.Topology.decoupled(4), params, cfg)
    want = None
    try:
        sp.integrate(sp.Topology.decoupled(4), params, cfg.with_overrides(backend="reference"))
    except sp.IntegrationDivergedError as exc:
        want = exc
    assert want is not None
    assert (info.value.oscillator, info.value.step) == (want.oscillator, want.step)


@pytest.mark.gpu
def test_reference_bench_lists_b200(plugged, capsys):
    import spinosc.cli as cli

    # the reference's default drift admission budget (1e-8 per 1e4 steps) rejects
    # its own numpy backend at these sizes (drift ~2e-6), so it is relaxed here
    rc = cli.main(["bench", "--n-list", "10,100", "--steps", "2000", "--backends",
                   "reference,gpu", "--repetitions", "1", "--drift-budget", "1e-2"])
    cap = capsys.readouterr()
    out = cap.out
    assert rc == 0, out + cap.err
    assert "gpu n=100:" in out


@pytest.mark.gpu
def test_reference_simulate_csv_byte_identical(plugged, tmp_path, capsys):
    """`spinosc simulate --backend gpu --output x.csv` (cli.py:171-187) through the
    whole-run hook: the trajectory CSV equals the one the reference's own
    `fused` backend writes for the same run, byte for byte."""
    import spinosc.cli as cli

    args = ["simulate", "--n", "60", "--steps", "400", "--record-stride", "40", "--seed", "3"]
    rc_gpu = cli.main(args + ["--backend", "gpu", "--output", str(tmp_path / "gpu.csv")])
    rc_ref = cli.main(args + ["--backend", "fused", "--output", str(tmp_path / "fused.csv")])
    out = capsys.readouterr().out
    assert rc_gpu == 0 and rc_ref == 0, out
    assert (tmp_path / "gpu.csv").read_bytes() == (tmp_path / "fused.csv").read_bytes()
    assert "backend=gpu n=60" in out


@pytest.mark.gpu
def test_reference_scaling_command_runs_b200(plugged, tmp_path, capsys):
    """`spinosc scaling --backend gpu` (cli.py:284-313): the reference's
    derivative-cost sweep times the B200 K0 derivative and fits an exponent
    (its fit needs four sizes spanning a decade, bench.py:233-239)."""
    import spinosc.cli as cli

    out_csv = tmp_path / "scaling.csv"
    rc = cli.main(["scaling", "--backend", "gpu", "--n-list", "100,300,1000,3000", "--evals", "3",
                   "--output", str(out_csv)])
    out = capsys.readouterr().out
    assert rc == 0, out
    assert "fitted scaling exponent" in out
    assert out_csv.read_text().splitlines()[0] == "n,seconds"


def test_elementwise_field_helpers_match_reference(plugged):
    """effective_field / spin_torque_strength: same operations as ref model.py:152-173."""
    import paper_2312_01121_b200 as sto

    g = np.random.default_rng(4)
    m = g.standard_normal((9, 3))
    m /= np.linalg.norm(m, axis=1, keepdims=True)
    for over in ({}, {"current": 3.1e-3, "h_appl": -120.0}):
        ours, ref = sto.PhysicalParams(**over), plugged.PhysicalParams(**over)
        assert np.array_equal(sto.effective_field(m, ours), plugged.effective_field(m, ref))
        assert np.array_equal(sto.spin_torque_strength(m, ours), plugged.spin_torque_strength(m, ref))


@pytest.mark.gpu
def test_total_b_matches_reference(plugged):
    """total_b with the coupling/input sums from the device pinned tree: bit-identical
    to the reference's numpy version (ref model.py:190-203)."""
    import paper_2312_01121_b200 as sto

    n = 37
    top_ref = plugged.build_topology(n, n_in=2, seed=5)
    top = sto.Topology(sto.CouplingMatrix(top_ref.coupling.entries),
                       sto.InputWeights(top_ref.input_weights.entries))
    g = np.random.default_rng(6)
    m = g.standard_normal((n, 3))
    m /= np.linalg.norm(m, axis=1, keepdims=True)
    u = g.uniform(-1, 1, 2)
    got = sto.total_b(m, u, top, sto.PhysicalParams())
    want = plugged.total_b(m, u, top_ref, plugged.PhysicalParams())
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


@pytest.mark.gpu
def test_coupling_field_plan_cached_and_bit_exact(plugged):
    """coupling_field_x on a CouplingMatrix reuses one device plan per matrix
    object (sto_plan_matvec, no W upload per call) and stays bit-identical to
    the reference's numpy pinned tree (ref model.py:176-180), also for a raw
    array (the one-shot path)."""
    import paper_2312_01121_b200 as sto
    from paper_2312_01121_b200 import model

    n = 300
    top_ref = plugged.build_topology(n, seed=9)
    cm = sto.CouplingMatrix(top_ref.coupling.entries)
    g = np.random.default_rng(10)
    before = len(model._MATVEC_PLANS)
    for _ in range(3):
        mx = g.uniform(-1, 1, n)
        got = sto.coupling_field_x(cm, mx, 0.7)
        want = plugged.coupling_field_x(top_ref.coupling, mx, 0.7)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
        raw = sto.coupling_field_x(top_ref.coupling.entries, mx, 0.7)
        assert np.array_equal(raw.view(np.uint64), want.view(np.uint64))
    assert len(model._MATVEC_PLANS) == before + 1


@pytest.mark.gpu
def test_integration_md_ctypes_stub_runs(plugged):
    """the ctypes stub a spinosc maintainer would paste -- executed
    verbatim (library path substituted) and checked against spinosc's own fused backend."""
    import re

    from conftest import ROOT

    text = (ROOT / "INTEGRATION.md").read_text()
    sec = text[text.index("## 3. Bind the C ABI directly"):]
    code = re.search(r"```python\n(.*?)```", sec, re.S).group(1)
    lib = str(ROOT / "paper_2312_01121_b200" / "libsto_b200.so")
    code = code.replace('ctypes.CDLL("libsto_b200.so")', f'ctypes.CDLL("{lib}")')
    ns: dict = {}
    exec(compile(code, "INTEGRATION.md", "exec"), ns)
    sp = plugged
    top = sp.build_topology(150, seed=2)
    params = sp.PhysicalParams()
    be = ns["StoBackend"](top, params)
    m = sp.initial_state(150)
    states = be.integrate_run(m, np.zeros((1, 1)), 1, 1e-11, 300, 100)
    want = sp.integrate(top, params, sp.RunConfig(n=150, steps=300, dt=1e-11, record_stride=100,
                                                  backend="fused"), backend=None)
    assert np.array_equal(states.view(np.uint64), want.states.view(np.uint64))
