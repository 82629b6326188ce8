"""Parity of the CUDA path with the reference, on a B200.

Bar: BIT-EXACT (uint64 view equality) for every single-trajectory kernel
family -- the reference's pinned operation order makes that achievable
(SURVEY §8(c)). Inputs are the golden fixtures the reference produced
(tests/golden/) and, for sizes without fixtures, the pinned CPU oracle
(oracle/sto_oracle.c, itself checked bit-for-bit against the reference in
tests/test_oracle.py) on the same seeded W, drive and initial state.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import assert_bit_equal, golden_trajectories, load_golden

pytestmark = pytest.mark.gpu

FORCE = {"auto": 0, "tiny": 0, "single": 0x4 | 0x8, "resident": 0x2 | 0x8, "stream": 0x1 | 0x8,
         "reg": 0x10 | 0x8, "cluster": 0x40 | 0x8}


@pytest.fixture(scope="module")
def sto():
    import paper_2312_01121_b200 as sto

    assert sto.available_backend_ids() == ["gpu"], "B200 backend not available"
    return sto


def _topology(sto, d):
    return sto.Topology(sto.CouplingMatrix(d["w"]), sto.InputWeights(d["w_in"]))


def _run(sto, d, family="auto"):
    from paper_2312_01121_b200.backends.b200 import B200Backend

    backend = B200Backend(_topology(sto, d), None, device=0, flags=FORCE[family],
                          consts=d["consts"])
    m = d["m0"].copy()
    states = backend.integrate_run(m, d["samples"], int(d["steps_per_sample"]), float(d["dt"]),
                                   int(d["steps"]), int(d["stride"]))
    return states, m, backend.plan_info


def _families(n):
    fams = ["auto", "stream", "resident"]
    if n <= 1024:
        fams.append("reg")
    if n <= 256:
        fams.append("cluster")
    if n <= 32:
        fams.append("tiny")
    if n <= 128:
        fams.append("single")
    return fams


@pytest.mark.parametrize("name", golden_trajectories())
def test_golden_trajectories_all_kernel_families(sto, name):
    d = load_golden(name)
    n = d["w"].shape[0]
    for fam in _families(n):
        if bool(d["diverged"]):
            with pytest.raises(sto.IntegrationDivergedError) as info:
                _run(sto, d, fam)
            assert (info.value.oscillator, info.value.step) == (int(d["bad_oscillator"]),
                                                               int(d["bad_step"])), fam
            continue
        states, final, info = _run(sto, d, fam)
        assert_bit_equal(states, d["states"], f"{name} [{fam}: {info['kernel_name']}]")
        assert_bit_equal(final, d["states"][-1], f"{name} final [{fam}]")


def test_public_integrate_matches_golden_config1(sto):
    """Config 1 (N=100, 1e4 steps, random drive) through the public API."""
    d = load_golden("traj_n100_cfg1.npz")
    top = _topology(sto, d)
    series = sto.InputSeries(d["samples"], int(d["steps_per_sample"]))
    cfg = sto.RunConfig(n=100, steps=int(d["steps"]), dt=float(d["dt"]),
                        record_stride=int(d["stride"]), input_series=series)
    traj = sto.integrate(top, sto.PhysicalParams(), cfg)
    assert_bit_equal(traj.states, d["states"], "config 1")
    assert traj.max_norm_drift == pytest.approx(float(d["drift"]), rel=0, abs=0)


@pytest.mark.parametrize("n", [33, 64, 65, 200, 257, 511, 513, 1000, 1025, 2049, 3000])
def test_oracle_parity_sizes(sto, oracle_mod, n):
    g = np.random.default_rng(n)
    w = g.uniform(-1, 1, (n, n)) / np.sqrt(n)
    np.fill_diagonal(w, 0.0)
    w_in = g.uniform(-1, 1, (n, 2))
    steps, stride, sps = 60, 7, 3
    samples = g.uniform(-1, 1, (20, 2))
    consts = sto.kernel_scalars(sto.PhysicalParams())
    m0 = sto.initial_state(n)
    want, _ = oracle_mod.integrate(w, w_in, consts, m0, samples, sps, 1e-11, steps, stride)
    d = dict(w=w, w_in=w_in, consts=np.array(consts), m0=m0, samples=samples,
             steps_per_sample=sps, dt=1e-11, steps=steps, stride=stride)
    for fam in _families(n):
        try:
            states, _, info = _run(sto, d, fam)
        except sto.ParameterError:
            continue  # family does not fit this size (e.g. resident at large n)
        assert_bit_equal(states, want, f"n={n} [{fam}: {info['kernel_name']}]")


def test_large_n_streaming_against_oracle(sto, oracle_mod):
    """N = 1e4 (the bench workload) over 3 steps, W streamed from HBM."""
    n = 10_000
    g = np.random.default_rng(10)
    w = (g.uniform(-1, 1, (n, n)) * (1.0 / np.sqrt(n))).astype(np.float64)
    np.fill_diagonal(w, 0.0)
    w_in = g.uniform(-1, 1, (n, 1))
    consts = sto.kernel_scalars(sto.PhysicalParams())
    m0 = sto.initial_state(n)
    samples = np.zeros((1, 1))
    want, _ = oracle_mod.integrate(w, w_in, consts, m0, samples, 1, 1e-11, 3, 1)
    d = dict(w=w, w_in=w_in, consts=np.array(consts), m0=m0, samples=samples,
             steps_per_sample=1, dt=1e-11, steps=3, stride=1)
    states, _, info = _run(sto, d, "auto")
    assert info["kernel_name"] == "stream"
    assert_bit_equal(states, want, "n=1e4")


def test_benched_config4_full_horizon_bit_exact(sto, oracle_mod):
    """configs[4] as benched (bench.py n1e4): N = 1e4, seed-0 reservoir (device
    build, as bench.py uses for large N), 1e3 RK4 steps -- the whole benched
    horizon, every 100th state bit-identical to the oracle (W streamed from
    HBM with the L2-resident slice).  ~1 min of 16-thread oracle time."""
    n, steps, stride = 10_000, 1000, 100
    top = sto.build_topology_device(n, seed=0)
    params = sto.PhysicalParams()
    cfg = sto.RunConfig(n=n, steps=steps, dt=1e-11, record_stride=stride)
    tr = sto.integrate(top, params, cfg)
    want, _ = oracle_mod.integrate(top.coupling.entries, top.input_weights.entries,
                                   sto.kernel_scalars(params), sto.initial_state(n),
                                   np.zeros((1, 1)), 1, 1e-11, steps, stride)
    assert_bit_equal(tr.states, want, "configs[4] n=1e4, 1e3 steps")


def test_benched_n4e4_full_horizon_bit_exact(sto, oracle_mod):
    """configs[4] upper end as benched (bench.py n4e4): N = 4e4, device-built
    seed-0 reservoir, 50 RK4 steps -- the chunked-x streaming kernel over the
    whole benched horizon, every 10th state bit-identical to the oracle
    (~45 s of 16-thread oracle time)."""
    n, steps, stride = 40_000, 50, 10
    top = sto.build_topology_device(n, seed=0)
    params = sto.PhysicalParams()
    cfg = sto.RunConfig(n=n, steps=steps, dt=1e-11, record_stride=stride)
    tr = sto.integrate(top, params, cfg)
    want, _ = oracle_mod.integrate(top.coupling.entries, top.input_weights.entries,
                                   sto.kernel_scalars(params), sto.initial_state(n),
                                   np.zeros((1, 1)), 1, 1e-11, steps, stride)
    assert_bit_equal(tr.states, want, "configs[4] n=4e4, 50 steps")


def test_derivative_golden(sto):
    from paper_2312_01121_b200.backends.b200 import B200Backend

    z = load_golden("deriv.npz")
    for key in sorted(k[:-2] for k in z if k.endswith("_m")):
        n, n_in, seed = (int(t.lstrip("ins")) for t in key.split("_"))
        t = load_golden(f"topo_n{n}_in{n_in}_s{seed}.npz")
        top = sto.Topology(sto.CouplingMatrix(t["w"]), sto.InputWeights(t["w_in"]))
        be = B200Backend(top, sto.PhysicalParams())
        out = np.empty((n, 3))
        be.derivative(z[key + "_m"], z[key + "_u"], out)
        assert_bit_equal(out, z[key + "_out"], f"derivative {key}")
        # the model-level function uses the same kernel
        got = sto.llg_derivative(z[key + "_m"], z[key + "_u"], top, sto.PhysicalParams())
        assert_bit_equal(got, z[key + "_out"], f"llg_derivative {key}")


def test_llg_derivative_consts_and_plan_cache(sto, oracle_mod):
    """model.llg_derivative honours a caller-supplied DerivedConstants (ref
    model.py:206-230) and reuses one device plan per (topology, scalars)."""
    from paper_2312_01121_b200 import model

    n = 300
    top = sto.build_topology(n, seed=4)
    p0, p1 = sto.PhysicalParams(), sto.PhysicalParams(current=2.5e-3)
    g = np.random.default_rng(4)
    m = g.normal(size=(n, 3))
    m /= np.linalg.norm(m, axis=1, keepdims=True)
    u = g.uniform(-1, 1, 1)
    want = oracle_mod.derivative(top.coupling.entries, top.input_weights.entries,
                                 sto.kernel_scalars(p1), m, u)
    got = sto.llg_derivative(m, u, top, p0, consts=sto.derive(p1))  # consts win over params
    assert_bit_equal(got, want, "llg_derivative(consts=)")
    before = len(model._BACKENDS[id(top)][1])
    for _ in range(3):
        again = sto.llg_derivative(m, u, top, p1)
    assert_bit_equal(again, want, "llg_derivative(params)")
    assert len(model._BACKENDS[id(top)][1]) == before  # same scalars: the cached plan


@pytest.mark.parametrize("n,n_in", [(33, 3), (500, 5), (3000, 2)])
def test_derivative_multichannel_against_oracle(sto, oracle_mod, n, n_in):
    """K0 (the reference plugin contract, derivative(m, u, out)) with n_in > 1:
    the input field is the pinned tree over the channels (cpu_jit.py:48-87)."""
    from paper_2312_01121_b200.backends.b200 import B200Backend

    g = np.random.default_rng(n)
    w = g.uniform(-1, 1, (n, n)) / np.sqrt(n)
    np.fill_diagonal(w, 0.0)
    w_in = g.uniform(-1, 1, (n, n_in))
    top = sto.Topology(sto.CouplingMatrix(w), sto.InputWeights(w_in))
    m = g.normal(size=(n, 3))
    m /= np.linalg.norm(m, axis=1, keepdims=True)
    u = g.uniform(-1, 1, n_in)
    be = B200Backend(top, sto.PhysicalParams())
    out = np.empty((n, 3))
    be.derivative(m, u, out)
    want = oracle_mod.derivative(w, w_in, sto.kernel_scalars(sto.PhysicalParams()), m, u)
    assert_bit_equal(out, want, f"K0 n={n} n_in={n_in}")


def test_derivative_on_device_tensors(sto):
    import torch

    from paper_2312_01121_b200.backends.b200 import B200Backend

    z = load_golden("deriv.npz")
    t = load_golden("topo_n100_in1_s0.npz")
    top = sto.Topology(sto.CouplingMatrix(t["w"]), sto.InputWeights(t["w_in"]))
    be = B200Backend(top, sto.PhysicalParams())
    m = torch.as_tensor(z["n100_in1_s0_m"], device="cuda")
    u = torch.as_tensor(z["n100_in1_s0_u"], device="cuda")
    out = torch.empty_like(m)
    be.derivative(m, u, out)
    torch.cuda.synchronize()
    assert_bit_equal(out.cpu().numpy(), z["n100_in1_s0_out"], "device-tensor derivative")


def test_tree_reduce_rows_golden(sto):
    z = load_golden("tree.npz")
    for i, w in enumerate(z["widths"]):
        rows = z["values"][z["offsets"][i]:z["offsets"][i + 1]].reshape(3, w)
        got = sto.tree_reduce_rows(rows)
        assert_bit_equal(got, z["sums"][3 * i:3 * i + 3], f"tree width {w}")


def test_decoupled_reproduces_single_oscillator(sto):
    """Reference acceptance A9: N=10 with W=0, u=0 equals N=1 bit-exactly."""
    p = sto.PhysicalParams()
    t10 = sto.integrate(sto.Topology.decoupled(10), p, sto.RunConfig(n=10, steps=1000, dt=1e-11))
    t1 = sto.integrate(sto.Topology.decoupled(1), p, sto.RunConfig(n=1, steps=1000, dt=1e-11))
    for k in range(10):
        assert_bit_equal(t10.states[:, k, :], t1.states[:, 0, :], f"row {k}")


def test_repeated_runs_identical(sto):
    top = sto.build_topology(300, seed=4)
    be = sto.create_backend("gpu", top, sto.PhysicalParams())
    cfg = sto.RunConfig(n=300, steps=100, dt=1e-11, record_stride=10)
    a = sto.integrate(top, sto.PhysicalParams(), cfg, backend=be)
    b = sto.integrate(top, sto.PhysicalParams(), cfg, backend=be)
    assert_bit_equal(a.states, b.states)


def test_host_buffer_abi_entry_point(sto, oracle_mod):
    """sto_integrate_host: the C-ABI call with HOST buffers (the e2e path)."""
    import ctypes

    from paper_2312_01121_b200 import _native

    d = load_golden("traj_n13.npz")
    plan = _native.Plan(d["w"], d["w_in"], d["consts"], device=0)
    m = d["m0"].copy()
    nrec = _native.n_records(int(d["steps"]), int(d["stride"]))
    states = np.empty((nrec, 13, 3))
    st = _native.Status()
    P = ctypes.POINTER(ctypes.c_double)
    rc = _native.lib().sto_integrate_host(plan._h, m.ctypes.data_as(P),
                                          d["samples"].ctypes.data_as(P), d["samples"].shape[0],
                                          int(d["steps_per_sample"]), float(d["dt"]),
                                          int(d["steps"]), int(d["stride"]),
                                          states.ctypes.data_as(P), ctypes.byref(st))
    assert rc == 0, _native.last_error()
    assert_bit_equal(states, d["states"])
    assert_bit_equal(m, d["states"][-1])


@pytest.mark.parametrize("warps", ["auto", "16", "20"])
def test_streaming_warp_counts_bit_exact(sto, oracle_mod, monkeypatch, warps):
    """The HBM-streaming kernel runs 20 warps per CTA when x fits one window
    (host: stream_threads) and 16 otherwise; both counts split the same
    (row, block) tree nodes, so the bits must not change (N = 5000, W 200 MB)."""
    if warps != "auto":
        monkeypatch.setenv("STO_GRID_WARPS", warps)
    n = 5000
    g = np.random.default_rng(5000)
    w = g.uniform(-1, 1, (n, n)) / np.sqrt(n / 3.0)
    np.fill_diagonal(w, 0.0)
    w_in = g.uniform(-1, 1, (n, 1))
    consts = sto.kernel_scalars(sto.PhysicalParams())
    m0 = sto.initial_state(n)
    samples = g.uniform(-1, 1, (4, 1))
    want, _ = oracle_mod.integrate(w, w_in, consts, m0, samples, 1, 1e-11, 4, 2)
    d = dict(w=w, w_in=w_in, consts=np.array(consts), m0=m0, samples=samples,
             steps_per_sample=1, dt=1e-11, steps=4, stride=2)
    states, _, info = _run(sto, d, "auto")
    assert info["kernel_name"] == "stream"
    assert info["threads"] == (512 if warps == "16" else 640), info
    assert_bit_equal(states, want, f"n=5000 warps={warps}")


def _random_case(sto, n, seed, steps, stride, n_in=1, sps=1, scale=None):
    g = np.random.default_rng(seed)
    w = g.random((n, n))
    w *= 2.0
    w -= 1.0
    w *= 1.0 / np.sqrt(n / 3.0) if scale is None else scale
    np.fill_diagonal(w, 0.0)
    w_in = g.uniform(-1, 1, (n, n_in))
    samples = g.uniform(-1, 1, (-(-steps // sps), n_in))
    return dict(w=w, w_in=w_in, consts=np.array(sto.kernel_scalars(sto.PhysicalParams())),
                m0=sto.initial_state(n), samples=samples, steps_per_sample=sps, dt=1e-11,
                steps=steps, stride=stride)


@pytest.mark.parametrize("n,chunk", [(3000, 1024), (5000, 512), (5000, 1024), (5000, 2048),
                                     (9000, 2048), (9000, 4096)])
def test_chunked_x_windows_bit_exact(sto, oracle_mod, monkeypatch, n, chunk):
    """The streaming kernel's chunked block loop (x staged in several shared-memory
    windows: per-chunk staging, bfirst / bcount, x_base offsets) -- the path every
    N >~ 2.4e4 run takes -- forced at small N with STO_CHUNK_COLS: bit-exact vs the
    oracle for the L2 (N = 3000) and HBM-streaming (N >= 5000) variants, whole
    run and a single derivative (K0)."""
    monkeypatch.setenv("STO_CHUNK_COLS", str(chunk))
    d = _random_case(sto, n, 7 * n + chunk, steps=5, stride=2, n_in=2, sps=2)
    want, _ = oracle_mod.integrate(d["w"], d["w_in"], d["consts"], d["m0"], d["samples"], 2,
                                   1e-11, 5, 2)
    states, final, info = _run(sto, d, "stream")
    assert info["kernel_name"] == "stream"
    assert info["x_window_cols"] == chunk and -(-info["ldw"] // chunk) >= 2, info
    assert_bit_equal(states, want, f"n={n} chunk={chunk}")
    assert_bit_equal(final, want[-1], "final")

    from paper_2312_01121_b200.backends.b200 import B200Backend

    top = _topology(sto, d)
    be = B200Backend(top, None, device=0, consts=d["consts"])
    m = np.random.default_rng(n).standard_normal((n, 3))
    u = np.array([0.3, -0.7])
    out = np.empty((n, 3))
    be.derivative(m, u, out)
    assert_bit_equal(out, oracle_mod.derivative(d["w"], d["w_in"], d["consts"], m, u,
                                                threads=oracle_mod.default_threads()),
                     f"derivative n={n} chunk={chunk}")


def test_n3e4_chunked_streaming_against_oracle(sto, oracle_mod):
    """N = 3e4 (W 7.2 GB): the real chunked-x configuration of configs[4]'s upper
    half (x = 2 windows of 16384 columns, chosen by the host, no knob), 2 RK4
    steps, bit-exact vs the oracle."""
    n = 30_000
    d = _random_case(sto, n, 30, steps=2, stride=1)
    d["samples"] = np.zeros((1, 1))
    want, _ = oracle_mod.integrate(d["w"], d["w_in"], d["consts"], d["m0"], d["samples"], 1,
                                   1e-11, 2, 1)
    states, final, info = _run(sto, d, "auto")
    assert info["kernel_name"] == "stream"
    assert info["x_window_cols"] < info["ldw"], info
    assert_bit_equal(states, want, "n=3e4")
    assert_bit_equal(final, want[-1], "n=3e4 final")


def test_register_kernel_epoch_wrap(sto, oracle_mod, monkeypatch):
    """The register kernel's LL exchange counts 31-bit epochs (bit 31 is the stop
    bit); runs longer than 2^29 RK4 steps wrap it.  STO_REG_EPOCH0 starts the
    count 16 stages before the wrap: the run must stay bit-exact (a counter that
    reached bit 31 would never match again and hang the kernel)."""
    monkeypatch.setenv("STO_REG_EPOCH0", str(0x7FFFFFF0))
    d = _random_case(sto, 1000, 1000, steps=30, stride=7)
    want, _ = oracle_mod.integrate(d["w"], d["w_in"], d["consts"], d["m0"], d["samples"], 1,
                                   1e-11, 30, 7)
    states, _, info = _run(sto, d, "reg")
    assert info["kernel_name"] == "reg"
    assert_bit_equal(states, want, "epoch wrap")


@pytest.mark.parametrize("n,split,sps,stride", [(100, 500, 1, 100), (100, 501, 3, 167),
                                               (1000, 60, 4, 20), (3000, 7, 2, 7)])
def test_resume_on_device_bit_exact(sto, oracle_mod, n, split, sps, stride):
    """f4 on the B200 path: run(a + b) == run(a) + resume(b) bit for bit (split
    inside a drive hold for 501 % 3), through the cluster / register /
    streaming kernels, and equal to the oracle."""
    total = 2 * split + (3 if split % 2 else 0)
    top = sto.build_topology(n, seed=n + split)
    p = sto.PhysicalParams()
    g = np.random.default_rng(split)
    full = sto.InputSeries(g.uniform(-1, 1, (-(-total // sps), 1)), sps)
    head = sto.InputSeries(full.samples[:-(-split // sps)], sps)
    whole = sto.integrate(top, p, sto.RunConfig(n=n, steps=total, dt=1e-11, record_stride=stride,
                                                input_series=full))
    first = sto.integrate(top, p, sto.RunConfig(n=n, steps=split, dt=1e-11, record_stride=stride,
                                                input_series=head))
    rest = sto.resume(first, top, p, total - split, input_series=full)
    assert_bit_equal(np.concatenate([first.states, rest.states[1:]]), whole.states, "resume")
    assert np.array_equal(np.concatenate([first.times, rest.times[1:]]), whole.times)
    want, _ = oracle_mod.integrate(top.coupling.entries, top.input_weights.entries,
                                   sto.kernel_scalars(p), sto.initial_state(n), full.samples, sps,
                                   1e-11, total, stride)
    assert_bit_equal(whole.states, want, "whole vs oracle")


@pytest.mark.parametrize("name,families", [("hz_n1_1e6.npz", ["auto", "single"]),
                                           ("hz_n1000_1e5.npz", ["auto", "stream"])])
def test_full_horizon_configs(sto, name, families):
    """configs[1] (N = 1, 1e6 RK4 steps) and configs[2] (N = 1000,
    build_topology(1000, seed=0), 1e5 steps) at the horizons BASELINE names,
    bit-exact against the reference's own trajectories (fixtures made by its
    numba engines), through the public integrate() and a second kernel family."""
    from conftest import horizon_topology

    d = load_golden(name)
    top = horizon_topology(d)
    n, steps, stride = int(d["n"]), int(d["steps"]), int(d["stride"])
    cfg = sto.RunConfig(n=n, steps=steps, dt=float(d["dt"]), record_stride=stride)
    traj = sto.integrate(top, sto.PhysicalParams(), cfg)
    assert_bit_equal(traj.states, d["states"], f"{name} public integrate")
    assert traj.max_norm_drift == float(d["drift"])
    dd = dict(w=top.coupling.entries, w_in=top.input_weights.entries, consts=d["consts"],
              m0=d["m0"], samples=np.zeros((1, 1)), steps_per_sample=1, dt=float(d["dt"]),
              steps=steps, stride=stride)
    for fam in families[1:]:
        states, _, info = _run(sto, dd, fam)
        assert_bit_equal(states, d["states"], f"{name} [{fam}: {info['kernel_name']}]")


@pytest.mark.parametrize("family", ["tiny", "cluster", "reg", "stream", "resident", "single"])
def test_runs_are_deterministic_and_stateless(sto, family):
    """SURVEY §5's determinism plan (the reference's thread-count / no-hidden-
    state tests, test_backends.py:104-135): the same run twice on one plan,
    and again after another plan of a different size ran in between, gives the
    same bits -- no state leaks between launches or plans."""
    from paper_2312_01121_b200.backends.b200 import B200Backend

    n = {"tiny": 20, "single": 100, "cluster": 100}.get(family, 200)
    g = np.random.default_rng(31)
    w = g.uniform(-1, 1, (n, n)) / np.sqrt(n)
    np.fill_diagonal(w, 0.0)
    top = sto.Topology(sto.CouplingMatrix(w), sto.InputWeights(g.uniform(-1, 1, (n, 1))))
    samples = g.uniform(-1, 1, (30, 1))
    be = B200Backend(top, sto.PhysicalParams(), flags=FORCE[family])

    def once(backend):
        m = sto.initial_state(n)
        return backend.integrate_run(m, samples, 2, 1e-11, 60, 10), m

    a, ma = once(be)
    b, mb = once(be)
    other = B200Backend(sto.build_topology(77, seed=2), sto.PhysicalParams())
    once_other = other.integrate_run(sto.initial_state(77), np.zeros((1, 1)), 1, 1e-11, 40, 40)
    assert np.isfinite(once_other).all()
    c, mc = once(be)
    assert_bit_equal(a, b, f"{family}: second run")
    assert_bit_equal(a, c, f"{family}: after another plan")
    assert_bit_equal(ma, mc, f"{family}: final state")
