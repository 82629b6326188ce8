"""Thread-block-cluster kernel (csrc/sto_cluster_kernel.cuh, 33 <= n <= 512 by
default): every cluster size K and W-columns-per-thread split C must reproduce
the pinned oracle BIT FOR BIT, including ragged row splits (n not a multiple
of P/K, so pad slots fall in every CTA), multi-channel drives held over several steps, recording strides, and
the reference's divergence report (integrator.py:174-177) -- all CTAs of the
cluster must stop after the same step with the same (oscillator, step).
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import assert_bit_equal, load_golden

pytestmark = pytest.mark.gpu

CLUSTER = 0x40 | 0x8  # STO_PLAN_FORCE_CLUSTER | STO_PLAN_NO_TINY


@pytest.fixture(autouse=True, params=[1, 0], ids=["teams-finish-rows", "owner-warp"])
def clu_variant(request, monkeypatch):
    """Every test runs on both cluster kernels (STO_CLU_HYB): clu_hyb_kernel
    (the teams run the RHS of their rows) and clu_rk4_kernel (owner warp)."""
    monkeypatch.setenv("STO_CLU_HYB", str(request.param))
    return request.param


def _variants(n):
    """(K, C) pairs the host accepts (sto_b200.cu): K a power of two, SEG = P/K <= 32
    rows per CTA, one owner warp + SEG*T GEMV threads within the launch bound."""
    pc = max(64, 1 << (max(n, 1) - 1).bit_length())
    out = []
    for c in (64, 32, 16):
        t = pc // c
        for k in (2, 4, 8, 16):
            seg = pc // k
            threads = 32 + 32 * (-(-seg * t // 32))
            if (1 <= t <= 32 and seg <= 32 and threads <= (576 if c == 16 else 288)
                    and (c != 64 or t == 8)):
                out.append((k, c))
    return out


def _backend(sto, top, monkeypatch, k, c, params=None, consts=None):
    from paper_2312_01121_b200.backends.b200 import B200Backend

    monkeypatch.setenv("STO_CLU_K", str(k))
    monkeypatch.setenv("STO_CLU_C", str(c))
    be = B200Backend(top, params, device=0, flags=CLUSTER, consts=consts)
    info = be.plan_info
    assert info["kernel_name"] == "cluster" and info["grid"] == k, info
    return be


@pytest.mark.parametrize("n,n_in", [(33, 1), (64, 3), (100, 1), (129, 2), (200, 1), (256, 2),
                                     (257, 1), (400, 2), (512, 1)])
def test_every_cluster_shape_bit_exact(monkeypatch, oracle_mod, n, n_in):
    """Rows are owned by x-position segments, so ragged n leaves pad slots in
    every CTA; all of them must still give the pinned tree's bits."""
    import paper_2312_01121_b200 as sto

    g = np.random.default_rng(1000 + n)
    w = g.uniform(-1, 1, (n, n)) / np.sqrt(n / 3.0)
    np.fill_diagonal(w, 0.0)
    w_in = g.uniform(-1, 1, (n, n_in))
    top = sto.Topology(sto.CouplingMatrix(w), sto.InputWeights(w_in))
    params = sto.PhysicalParams()
    consts = sto.kernel_scalars(params)
    steps, sps, stride = 61, 4, 6
    samples = g.uniform(-1, 1, (16, n_in))
    m0 = sto.initial_state(n)
    want, _ = oracle_mod.integrate(w, w_in, consts, m0, samples, sps, 1e-11, steps, stride)
    variants = _variants(n)
    assert variants
    for k, c in variants:
        be = _backend(sto, top, monkeypatch, k, c, params)
        m = m0.copy()
        got = be.integrate_run(m, samples, sps, 1e-11, steps, stride)
        assert_bit_equal(got, want, f"n={n} K={k} C={c}")
        assert_bit_equal(m, want[-1], f"n={n} K={k} C={c} final state")
        be.close()


@pytest.mark.parametrize("name", ["traj_n6_diverge.npz", "traj_n6_diverge_late.npz"])
def test_divergence_reported_by_every_cluster_size(monkeypatch, name):
    import paper_2312_01121_b200 as sto

    d = load_golden(name)
    top = sto.Topology(sto.CouplingMatrix(d["w"]), sto.InputWeights(d["w_in"]))
    for k in (2, 4, 8, 16):
        be = _backend(sto, top, monkeypatch, k, 32, consts=d["consts"])
        with pytest.raises(sto.IntegrationDivergedError) as info:
            be.integrate_run(d["m0"].copy(), d["samples"], int(d["steps_per_sample"]),
                             float(d["dt"]), int(d["steps"]), int(d["stride"]))
        assert (info.value.oscillator, info.value.step) == (int(d["bad_oscillator"]),
                                                           int(d["bad_step"])), k
        be.close()


@pytest.mark.parametrize("stride", [1, 3, 7, 70])
@pytest.mark.parametrize("hyb", ["1", "0"])
def test_divergence_between_stop_flag_rounds(monkeypatch, oracle_mod, stride, hyb):
    """The cluster stops on stop-flag rounds (at most one per kCluFlagEvery = 64
    steps), not on every recording step: a row that goes non-finite between
    rounds is still reported at ITS recording step, first oscillator first
    (integrator.py:174-177), and the run stops on the next round.  Late
    divergence of traj_n6_diverge_late's reservoir, embedded in n = 100 / 200
    (the other rows decoupled), at record strides that put it between rounds."""
    import paper_2312_01121_b200 as sto

    d = load_golden("traj_n6_diverge_late.npz")
    monkeypatch.setenv("STO_CLU_HYB", hyb)
    n = 100 if hyb == "1" else 200
    w = np.zeros((n, n))
    w[:6, :6] = d["w"]
    w_in = np.zeros((n, 1))
    w_in[:6] = d["w_in"]
    top = sto.Topology(sto.CouplingMatrix(w), sto.InputWeights(w_in))
    m0 = sto.initial_state(n)
    m0[:6] = d["m0"]
    steps, sps = int(d["steps"]), int(d["steps_per_sample"])
    with pytest.raises(oracle_mod.OracleDiverged) as want:
        oracle_mod.integrate(w, w_in, d["consts"], m0, d["samples"], sps, float(d["dt"]), steps,
                             stride)
    for k in (2, 8):
        if (k, 32) not in _variants(n):
            continue
        be = _backend(sto, top, monkeypatch, k, 32, consts=d["consts"])
        with pytest.raises(sto.IntegrationDivergedError) as info:
            be.integrate_run(m0.copy(), d["samples"], sps, float(d["dt"]), steps, stride)
        assert (info.value.oscillator, info.value.step) == (want.value.oscillator,
                                                           want.value.step), (k, stride)
        be.close()


def test_golden_config1_through_cluster(monkeypatch):
    """configs[0] (N = 100, 1e4 steps, a new drive sample every step): the
    reference's own trajectory, every cluster size."""
    import paper_2312_01121_b200 as sto

    d = load_golden("traj_n100_cfg1.npz")
    top = sto.Topology(sto.CouplingMatrix(d["w"]), sto.InputWeights(d["w_in"]))
    for k, c in _variants(100):
        be = _backend(sto, top, monkeypatch, k, c, consts=d["consts"])
        got = be.integrate_run(d["m0"].copy(), d["samples"], int(d["steps_per_sample"]),
                               float(d["dt"]), int(d["steps"]), int(d["stride"]))
        assert_bit_equal(got, d["states"], f"config 1 K={k} C={c}")
        be.close()


def test_auto_selects_cluster_for_small_reservoirs():
    import paper_2312_01121_b200 as sto
    from paper_2312_01121_b200.backends.b200 import B200Backend

    for n, want in [(32, "tiny"), (33, "cluster"), (256, "cluster"), (257, "cluster"), (512, "cluster"),
                    (513, "reg")]:
        g = np.random.default_rng(n)
        w = g.uniform(-1, 1, (n, n)) / np.sqrt(n)
        np.fill_diagonal(w, 0.0)
        top = sto.Topology(sto.CouplingMatrix(w), sto.InputWeights(g.uniform(-1, 1, (n, 1))))
        be = B200Backend(top, sto.PhysicalParams(), device=0)
        assert be.plan_info["kernel_name"] == want, (n, be.plan_info)
        be.close()


def test_repeated_launches_identical(monkeypatch):
    """mbarrier phases and buffers are re-initialised per launch: back-to-back
    runs on one plan give identical bits."""
    import paper_2312_01121_b200 as sto

    n = 150
    g = np.random.default_rng(5)
    w = g.uniform(-1, 1, (n, n)) / np.sqrt(n)
    np.fill_diagonal(w, 0.0)
    top = sto.Topology(sto.CouplingMatrix(w), sto.InputWeights(g.uniform(-1, 1, (n, 1))))
    be = _backend(sto, top, monkeypatch, 8, 32, sto.PhysicalParams())
    drive = g.uniform(-1, 1, (500, 1))
    runs = [be.integrate_run(sto.initial_state(n), drive, 1, 1e-11, 500, 50) for _ in range(4)]
    for r in runs[1:]:
        assert_bit_equal(r, runs[0], "repeat")
    be.close()
