"""The CPU oracle (oracle/sto_oracle.c) pinned against the reference's outputs.

Every fixture in tests/golden/ was produced by the reference package itself
(tests/golden/make_golden.py); the oracle must reproduce each one bit for
bit before it is trusted as the parity checker of the CUDA path.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import assert_bit_equal, golden_trajectories, load_golden


def test_tree_sums_bit_exact(oracle_mod):
    z = load_golden("tree.npz")
    for i, w in enumerate(z["widths"]):
        rows = z["values"][z["offsets"][i]:z["offsets"][i + 1]].reshape(3, w)
        got = np.array([oracle_mod.tree_sum(r) for r in rows])
        assert_bit_equal(got, z["sums"][3 * i:3 * i + 3], f"tree width {w}")


def test_derivatives_bit_exact(oracle_mod):
    z = load_golden("deriv.npz")
    keys = sorted(k[:-2] for k in z if k.endswith("_m"))
    assert keys
    for key in keys:
        n, n_in, seed = (int(t[1:]) if t[0] in "ns" else int(t[2:])
                         for t in key.split("_"))
        topo = load_golden(f"topo_n{n}_in{n_in}_s{seed}.npz")
        for threads in (1, 3):
            got = oracle_mod.derivative(topo["w"], topo["w_in"], z["consts"], z[key + "_m"],
                                        z[key + "_u"], threads=threads)
            assert_bit_equal(got, z[key + "_out"], f"derivative {key} threads={threads}")


@pytest.mark.parametrize("threads", [1, 2], ids=["serial", "openmp"])
@pytest.mark.parametrize("name", golden_trajectories())
def test_trajectories_bit_exact(oracle_mod, name, threads):
    """Both oracle paths (single thread: no OpenMP constructs; several threads:
    one parallel region per run) against the reference's own trajectories."""
    d = load_golden(name)
    args = (d["w"], d["w_in"], d["consts"], d["m0"], d["samples"],
            int(d["steps_per_sample"]), float(d["dt"]), int(d["steps"]), int(d["stride"]))
    if bool(d["diverged"]):
        with pytest.raises(oracle_mod.OracleDiverged) as info:
            oracle_mod.integrate(*args, threads=threads)
        assert (info.value.oscillator, info.value.step) == (int(d["bad_oscillator"]),
                                                           int(d["bad_step"]))
        return
    states, final = oracle_mod.integrate(*args, threads=threads)
    assert_bit_equal(states, d["states"], name)
    assert_bit_equal(final, d["states"][-1], name + " final")


def test_thread_count_does_not_change_bits(oracle_mod):
    d = load_golden("traj_n160_params.npz")
    runs = [oracle_mod.integrate(d["w"], d["w_in"], d["consts"], d["m0"], d["samples"], 1,
                                 float(d["dt"]), 40, 10, threads=t)[0] for t in (1, 2, 5)]
    assert_bit_equal(runs[1], runs[0])
    assert_bit_equal(runs[2], runs[0])


def test_signed_zero_carry(oracle_mod):
    # odd tail carried unchanged: -0.0 must survive (padding with +0.0 would not)
    assert np.signbit(oracle_mod.tree_sum([-0.0]))
    assert np.signbit(oracle_mod.tree_sum([-0.0, -0.0, -0.0]))
    assert not np.signbit(oracle_mod.tree_sum([-0.0, 0.0, -0.0]))


@pytest.mark.parametrize("name", ["hz_n1_1e6.npz", "hz_n1000_1e5.npz"])
def test_full_horizon_fixtures(oracle_mod, name):
    """BASELINE configs[1] (N = 1, 1e6 steps) and configs[2] (N = 1000, seed-0
    W, 1e5 steps) at their full horizons, as the reference's own numba engines
    produced them: the oracle must reproduce every recorded state."""
    from conftest import horizon_topology

    d = load_golden(name)
    top = horizon_topology(d)
    states, final = oracle_mod.integrate(top.coupling.entries, top.input_weights.entries,
                                         d["consts"], d["m0"], np.zeros((1, 1)), 1,
                                         float(d["dt"]), int(d["steps"]), int(d["stride"]))
    assert_bit_equal(states, d["states"], name)
