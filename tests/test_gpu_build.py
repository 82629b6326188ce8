"""Device reservoir construction against the host build.

* Draws: `sto_pcg64_fill` must reproduce `RngStream.uniform_pm1` (numpy's
  Generator(PCG64(seed)).random() mapped to 2u - 1, ref topology.py:48-54)
  bit for bit at any offset, and place the coupling draws row-major on the
  off-diagonal (ref :255-257).
* Normalisation: rho from the device Arnoldi matvecs agrees with the host
  restatement to 1e-12 relative (summation order differs; the reference's
  BLAS order is not pinned either), hence W to the same relative bound and
  W_in exactly.
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch

    return torch


@pytest.mark.parametrize("seed", [0, 7, 2**40 + 3])
@pytest.mark.parametrize("offset,count", [(0, 1), (0, 33), (5, 1000), (123457, 40000)])
def test_uniform_draws_bit_exact(torch, seed, offset, count):
    from paper_2312_01121_b200 import _native, RngStream

    out = torch.empty(count, dtype=torch.float64, device="cuda")
    _native.pcg64_fill(out, count, offset, _native.pcg64_words(seed))
    rs = RngStream(seed)
    if offset:
        rs.uniform_pm1(offset)
    want = rs.uniform_pm1(count)
    got = out.cpu().numpy()
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


@pytest.mark.parametrize("n", [2, 3, 7, 33, 100, 257])
def test_offdiagonal_placement(torch, n):
    from paper_2312_01121_b200 import _native, RngStream

    w = torch.full((n, n), 7.0, dtype=torch.float64, device="cuda")
    _native.pcg64_fill(w, n * (n - 1), 0, _native.pcg64_words(n), diag_n=n, ld=n)
    want = np.zeros((n, n))
    want[~np.eye(n, dtype=bool)] = RngStream(n).uniform_pm1(n * (n - 1))
    assert np.array_equal(w.cpu().numpy().view(np.uint64), want.view(np.uint64))


@pytest.mark.parametrize("n,n_in,seed", [(1, 1, 0), (2, 1, 1), (13, 2, 7), (100, 1, 0), (300, 3, 5),
                                         (1200, 1, 0)])
def test_device_topology_matches_host(n, n_in, seed):
    import paper_2312_01121_b200 as sto

    dev = sto.build_topology_device(n, n_in=n_in, seed=seed)
    host = sto.build_topology(n, n_in=n_in, seed=seed)
    assert np.array_equal(dev.input_weights.entries.view(np.uint64),
                          host.input_weights.entries.view(np.uint64))
    wd, wh = dev.coupling.entries, host.coupling.entries
    assert np.all(np.diagonal(wd) == 0.0)
    if n > 1:
        rho_h = sto.spectral_radius(wd * dev.coupling.rho)
        assert abs(dev.coupling.rho - rho_h) <= 1e-12 * rho_h
        assert np.max(np.abs(wd - wh)) <= 1e-12 * np.max(np.abs(wh))


def test_integrate_reads_device_coupling_in_place(oracle_mod):
    """A plan built from the device W gives the same trajectory bits as one built
    from the same W copied to the host (no hidden host round trip changes W)."""
    import paper_2312_01121_b200 as sto

    n, steps = 500, 100
    dev = sto.build_topology_device(n, seed=3)
    host = sto.Topology(sto.CouplingMatrix(dev.coupling.entries.copy()), dev.input_weights)
    cfg = sto.RunConfig(n=n, steps=steps, dt=1e-11, record_stride=25)
    a = sto.integrate(dev, sto.PhysicalParams(), cfg)
    b = sto.integrate(host, sto.PhysicalParams(), cfg)
    assert np.array_equal(a.states.view(np.uint64), b.states.view(np.uint64))
    want, _ = oracle_mod.integrate(host.coupling.entries, host.input_weights.entries,
                                   sto.kernel_scalars(sto.PhysicalParams()), sto.initial_state(n),
                                   np.zeros((1, 1)), 1, 1e-11, steps, 25)
    assert np.array_equal(a.states.view(np.uint64), want.view(np.uint64))
