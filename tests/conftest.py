"""Shared fixtures.  `gpu` marks tests that need a B200 (run on the GPU box)."""

from __future__ import annotations

import glob
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 GPU and libsto_b200.so")


def fuzz_examples(default: int) -> int:
    """Hypothesis examples per fuzz test: STO_FUZZ_SCALE multiplies the default
    (the long fuzz campaign of profiles/r02*_fuzz.log runs with a large scale)."""
    return max(1, int(default * float(os.environ.get("STO_FUZZ_SCALE", "1"))))


def load_golden(name: str) -> dict:
    with np.load(GOLDEN / name, allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def golden_trajectories() -> list[str]:
    return sorted(os.path.basename(p) for p in glob.glob(str(GOLDEN / "traj_*.npz")))


def bits(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64)).view(np.uint64)


def assert_bit_equal(got, want, what: str = "") -> None:
    got, want = np.asarray(got), np.asarray(want)
    assert got.shape == want.shape, f"{what}: shape {got.shape} vs {want.shape}"
    if not np.array_equal(bits(got), bits(want)):
        diff = np.abs(got - want)
        idx = np.unravel_index(np.nanargmax(np.where(np.isnan(diff), 0, diff)), diff.shape)
        nbad = int((bits(got) != bits(want)).sum())
        raise AssertionError(f"{what}: {nbad} values differ in bits; max |diff| "
                             f"{diff[idx]:.3e} at {idx}")


@pytest.fixture(scope="session")
def params():
    from paper_2312_01121_b200 import PhysicalParams

    return PhysicalParams()


@pytest.fixture(scope="session")
def oracle_mod():
    from oracle import oracle

    oracle.build()
    return oracle


@pytest.fixture(scope="session")
def spinosc_ref():
    """The reference package itself, installed offline into baseline/_ref (git-ignored,
    travels to the GPU box with the snapshot); tests using it skip when it is absent."""
    ref = ROOT / "baseline" / "_ref"
    if ref.is_dir() and str(ref) not in sys.path:
        sys.path.append(str(ref))
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_sto")
    return pytest.importorskip("spinosc")


def horizon_topology(d: dict):
    """build_topology(n, seed) for a full-horizon fixture (hz_*.npz, which stores
    only W's sha256 and the reference's rho): W = the seeded PCG64 draws / rho,
    the reference's own steps (topology.py:241-265) with rho taken from the
    fixture.  rho comes out of LAPACK (the Arnoldi eigensolve), whose bits
    depend on the host's BLAS build and CPU, so the GPU box must not recompute
    it; the draws and the elementwise IEEE division are portable.  The rebuilt
    W is refused unless its bits are the ones the reference integrated."""
    import hashlib

    from paper_2312_01121_b200 import CouplingMatrix, InputWeights, Topology
    from paper_2312_01121_b200.topology import RngStream

    n, rho = int(d["n"]), float(d["rho"])
    stream = RngStream(int(d["seed"]))
    w = np.zeros((n, n))
    if n > 1:
        w[~np.eye(n, dtype=bool)] = stream.uniform_pm1(n * (n - 1))
        w /= rho
    w_in = stream.uniform_pm1(n).reshape(n, 1)
    assert hashlib.sha256(w.tobytes()).hexdigest() == str(d["w_sha256"]), "W bits differ"
    assert hashlib.sha256(w_in.tobytes()).hexdigest() == str(d["w_in_sha256"]), "W_in differs"
    return Topology(CouplingMatrix(w), InputWeights(w_in))


HORIZONS = ["hz_n1_1e6.npz", "hz_n1000_1e5.npz"]
