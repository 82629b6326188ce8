"""Generate the golden fixtures in tests/golden/ from the REFERENCE package.

Run here (where /root/reference exists), never on the GPU box:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

It imports `spinosc` from /root/reference/pkg/src and records, with the
reference's own definitional backend ("reference", numpy) cross-checked
against "fused" (numba):
  tree.npz      pinned adjacent-pairs tree sums (model.tree_reduce_rows)
  topo_*.npz    build_topology(n, n_in, seed) coupling + input weights
  deriv.npz     single derivative evaluations at scrambled states
  traj_*.npz    whole integrate() runs: inputs, recorded states, or the
                IntegrationDivergedError location
The fixtures are what pins the C oracle (oracle/sto_oracle.c) and the CUDA
path; see tests/test_oracle.py and tests/test_gpu_parity.py.
"""

from __future__ import annotations

import math
import os
import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, str(REF_SRC))

import spinosc  # noqa: E402
from spinosc import (InputSeries, PhysicalParams, RunConfig, Topology,  # noqa: E402
                     build_topology, integrate)
from spinosc.backends.cpu_jit import _scalar_pack  # noqa: E402
from spinosc.model import tree_reduce_rows  # noqa: E402
from spinosc.topology import initial_state  # noqa: E402


def scrambled(n: int, seed: int) -> np.ndarray:
    g = np.random.default_rng(seed)
    m = g.standard_normal((n, 3))
    return m / np.linalg.norm(m, axis=1, keepdims=True)


def make_tree() -> None:
    widths = [1, 2, 3, 4, 5, 7, 8, 9, 17, 31, 32, 33, 63, 64, 65, 100, 127, 128, 129,
              255, 256, 257, 511, 513, 999, 1000, 1023, 1024, 1025, 2047, 2049, 4097]
    g = np.random.default_rng(2312)
    rows, sums, offsets = [], [], [0]
    for w in widths:
        block = g.standard_normal((3, w)) * np.exp(g.uniform(-20, 20, size=(3, w)))
        block[0, ::7] = -0.0          # signed zeros must survive the odd-tail carry
        out = np.empty(3)
        tree_reduce_rows(block.copy(), np.empty((3, (w + 1) // 2)), out)
        rows.append(block.ravel())
        sums.append(out)
        offsets.append(offsets[-1] + block.size)
    np.savez(OUT / "tree.npz", widths=np.array(widths), values=np.concatenate(rows),
             offsets=np.array(offsets), sums=np.concatenate(sums))


TOPOS = [(1, 1, 0), (2, 1, 1), (3, 1, 3), (6, 2, 5), (7, 1, 11), (13, 1, 7),
         (33, 3, 33), (100, 1, 0), (160, 1, 3)]


def make_topos() -> dict:
    tops = {}
    for n, n_in, seed in TOPOS:
        t = build_topology(n, n_in=n_in, seed=seed)
        tops[(n, n_in, seed)] = t
        np.savez(OUT / f"topo_n{n}_in{n_in}_s{seed}.npz", w=t.coupling.entries,
                 w_in=t.input_weights.entries)
    return tops


def make_deriv(tops: dict) -> None:
    params = PhysicalParams()
    rec = {}
    for (n, n_in, seed), t in tops.items():
        m = scrambled(n, seed + 100)
        u = np.linspace(-0.9, 0.7, n_in)
        outs = []
        for bid in ("reference", "fused"):
            out = np.empty((n, 3))
            spinosc.create_backend(bid, t, params).derivative(m, u, out)
            outs.append(out)
        assert np.array_equal(outs[0], outs[1])
        rec[f"n{n}_in{n_in}_s{seed}_m"] = m
        rec[f"n{n}_in{n_in}_s{seed}_u"] = u
        rec[f"n{n}_in{n_in}_s{seed}_out"] = outs[0]
    rec["consts"] = np.array(_scalar_pack(params))
    np.savez(OUT / "deriv.npz", **rec)


def run_case(name, topology, params, steps, dt, stride, series=None,
             check_fused=True) -> None:
    cfg = RunConfig(n=topology.n, steps=steps, dt=dt, record_stride=stride,
                    input_series=series, backend="reference")
    series = series if series is not None else InputSeries.zeros(topology.n_in)
    rec = dict(w=topology.coupling.entries, w_in=topology.input_weights.entries,
               consts=np.array(_scalar_pack(params)), m0=initial_state(topology.n),
               samples=series.samples, steps_per_sample=series.steps_per_sample,
               dt=dt, steps=steps, stride=stride)
    try:
        traj = integrate(topology, params, cfg)
        rec.update(states=traj.states, times=traj.times, drift=traj.max_norm_drift,
                   diverged=False)
        if check_fused:
            other = integrate(topology, params, cfg.with_overrides(backend="fused"))
            assert np.array_equal(other.states, traj.states), name
    except spinosc.IntegrationDivergedError as e:
        rec.update(diverged=True, bad_oscillator=e.oscillator, bad_step=e.step)
    np.savez(OUT / f"traj_{name}.npz", **rec)
    print(name, "diverged" if rec["diverged"] else f"drift={rec['drift']:.3e}")


def make_trajs(tops: dict) -> None:
    p = PhysicalParams()
    run_case("n1_free", tops[(1, 1, 0)], p, 20000, 1e-11, 1000)
    g = np.random.default_rng(7)
    run_case("n7_input", tops[(7, 1, 11)], p, 500, 1e-11, 50,
             InputSeries(g.uniform(-1, 1, (500, 1)), 1))
    run_case("n13", tops[(13, 1, 7)], p, 200, 1e-11, 20)
    run_case("n33_multi", tops[(33, 3, 33)], p, 398, 1e-11, 40,
             InputSeries(g.uniform(-1, 1, (100, 3)), 4))
    run_case("n100_cfg1", tops[(100, 1, 0)], p, 10000, 1e-11, 1000,
             InputSeries(np.random.default_rng(1).uniform(-1, 1, (10000, 1)), 1),
             check_fused=False)
    run_case("decoupled10", Topology.decoupled(10), p, 1000, 1e-11, 100)
    run_case("precession", Topology.decoupled(1),
             PhysicalParams(alpha=0.0, current=0.0, h_k=4.0 * math.pi * 1448.3),
             400, 1e-12, 40)
    run_case("n160_params", tops[(160, 1, 3)],
             PhysicalParams(alpha=0.01, current=3.0e-3, a_cp=2.0, a_in=0.5), 300,
             1e-11, 30, InputSeries(np.array([[0.3]]), 1))
    run_case("n6_diverge", tops[(6, 2, 5)],
             PhysicalParams(a_cp=1.0e9), 400, 2e-10, 10)
    # only oscillator 3 is driven, and only from step 55 on: the blow-up must be
    # reported at oscillator 3 on the first recording step after it happens
    from spinosc.topology import CouplingMatrix, InputWeights
    w_in = np.zeros((6, 1))
    w_in[3, 0] = 0.75
    late = Topology(CouplingMatrix.zeros(6), InputWeights(w_in))
    drive = np.zeros((20, 1))
    drive[11:] = 1.0e12
    run_case("n6_diverge_late", late, p, 100, 1e-11, 10, InputSeries(drive, 5))


def _reference_rho(n: int) -> float:
    """The reference's rho for build_topology(n, seed=0) (topology.py:241-265)."""
    from spinosc.topology import RngStream, spectral_radius

    if n == 1:
        return 0.0
    w = np.zeros((n, n))
    w[~np.eye(n, dtype=bool)] = RngStream(0).uniform_pm1(n * (n - 1))
    return float(spectral_radius(w))


def make_horizons() -> None:
    """BASELINE configs[1] and configs[2] at their FULL horizons, by the
    reference's own numba engines (bit-identical to "reference", A2):
      hz_n1_1e6.npz      N = 1, u = 0, 1e6 RK4 steps, recorded every 1e5
      hz_n1000_1e5.npz   N = 1000, build_topology(1000, seed=0), u = 0, 1e5
                         steps, recorded every 1e4
    W is not stored (8 MB): the consumer rebuilds it from the seeded draws
    divided by the stored `rho` and must first match `w_sha256` /
    `w_in_sha256`.  rho is stored because its bits depend on the LAPACK build
    and CPU behind the spectral radius; the GPU box's differs."""
    import hashlib

    p = PhysicalParams()
    for name, n, steps, stride, engine in (("hz_n1_1e6", 1, 1_000_000, 100_000, "fused"),
                                           ("hz_n1000_1e5", 1000, 100_000, 10_000, "parallel")):
        top = build_topology(n, n_in=1, seed=0)
        cfg = RunConfig(n=n, steps=steps, dt=1e-11, record_stride=stride, backend=engine)
        traj = integrate(top, p, cfg)
        w = np.ascontiguousarray(top.coupling.entries)
        w_in = np.ascontiguousarray(top.input_weights.entries)
        np.savez(OUT / f"{name}.npz", n=n, seed=0, steps=steps, stride=stride, dt=1e-11,
                 consts=np.array(_scalar_pack(p)), m0=initial_state(n),
                 w_sha256=hashlib.sha256(w.tobytes()).hexdigest(),
                 w_in_sha256=hashlib.sha256(w_in.tobytes()).hexdigest(),
                 rho=_reference_rho(n),
                 states=traj.states, times=traj.times, drift=traj.max_norm_drift,
                 engine=engine)
        print(name, f"drift={traj.max_norm_drift:.3e}", f"{traj.elapsed_seconds:.1f}s")


if __name__ == "__main__":
    if sys.argv[1:] == ["horizons"]:
        make_horizons()
        sys.exit(0)
    make_tree()
    tops = make_topos()
    make_deriv(tops)
    make_trajs(tops)
    make_horizons()
