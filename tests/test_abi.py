"""The C-ABI library loads and exports every entry point include/sto.h declares.

CPU-only: no compute call is made; only entry points that must work (and
fail cleanly) without a GPU are exercised.
"""

from __future__ import annotations

import ctypes
import re

import pytest

from conftest import ROOT

HEADER = ROOT / "include" / "sto.h"


def declared_functions() -> list[str]:
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sto_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def native():
    from paper_2312_01121_b200 import _native

    if not _native.LIB_PATH.exists():
        import __graft_entry__

        __graft_entry__.build()
    return _native


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ("sto_probe", "sto_plan_create", "sto_plan_destroy", "sto_derivative",
                     "sto_integrate", "sto_integrate_host", "sto_last_error"):
        assert required in names


def test_library_exports_every_declared_symbol(native):
    lib = ctypes.CDLL(str(native.LIB_PATH))
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, f"not exported: {missing}"
    # and the Python binding knows every one of them
    assert set(declared_functions()) == set(native.SIGNATURES)


def test_calls_that_need_no_gpu(native):
    lib = native.lib()
    assert lib.sto_abi_version() == 2
    assert lib.sto_n_records(10, 3) == 5
    assert lib.sto_n_records(10, 5) == 3
    assert lib.sto_n_records(0, 1) == 0


def test_probe_and_plan_fail_cleanly_without_gpu(native):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    assert native.probe(0) is False
    import numpy as np

    from paper_2312_01121_b200.errors import BackendUnavailableError

    with pytest.raises(BackendUnavailableError):
        native.Plan(np.zeros((2, 2)), np.zeros((2, 1)), [0.0] * 11, device=0)


def test_gpu_backend_refuses_cpu(params):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2312_01121_b200 as sto

    with pytest.raises(sto.BackendUnavailableError):
        sto.create_backend("gpu", sto.Topology.decoupled(1), params)
    with pytest.raises(sto.BackendUnavailableError):
        sto.run(sto.RunConfig(n=2, steps=1, dt=1e-11))
