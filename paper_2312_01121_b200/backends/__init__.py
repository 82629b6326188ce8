"""Backend registry: the reference's plugin API (`spinosc/backends/__init__.py`).

`register_backend / unregister_backend / list_backends /
available_backend_ids / create_backend` keep the reference's names,
arguments and error behaviour (`:43-85`): ids map to (kind, requires, probe,
factory); registration order is presentation order; replacing an id is
allowed; unknown or unavailable ids raise `BackendUnavailableError`
listing what is available; `probe` never raises.

This package registers exactly one backend, "gpu" -- the B200 persistent
kernel (backends/b200.py) in place of the reference's torch offload. It has
no CPU backends: the reference's "reference"/"fused"/"parallel" engines are
the oracle, not part of this product.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

from ..errors import BackendUnavailableError


@dataclass(frozen=True)
class BackendDescriptor:
    backend_id: str
    kind: str
    available: bool
    requires: str


@dataclass(frozen=True)
class _Registration:
    kind: str
    requires: str
    probe: Callable[[], bool]
    factory: Callable[..., object]


_REGISTRY: dict[str, _Registration] = {}


def _safe_probe(entry: _Registration) -> bool:
    try:
        return bool(entry.probe())
    except Exception:
        return False


def register_backend(backend_id: str, kind: str, requires: str,
                     probe: Callable[[], bool], factory: Callable[..., object]) -> None:
    """Add or replace a registration; factory(topology, params, workers=, gpu_device=)."""
    _REGISTRY[backend_id] = _Registration(kind, requires, probe, factory)


def unregister_backend(backend_id: str) -> None:
    _REGISTRY.pop(backend_id, None)


def list_backends() -> list[BackendDescriptor]:
    return [BackendDescriptor(bid, e.kind, _safe_probe(e), e.requires)
            for bid, e in _REGISTRY.items()]


def available_backend_ids() -> list[str]:
    return [bid for bid, e in _REGISTRY.items() if _safe_probe(e)]


def create_backend(backend_id: str, topology, params, *, workers: int | None = None,
                   gpu_device=None):
    entry = _REGISTRY.get(backend_id)
    if entry is None or not _safe_probe(entry):
        raise BackendUnavailableError(backend_id, available_backend_ids())
    return entry.factory(topology, params, workers=workers, gpu_device=gpu_device)


def _gpu_probe() -> bool:
    from .b200 import is_available

    return is_available()


def _gpu_factory(topology, params, workers=None, gpu_device=None):
    from .b200 import make_backend

    return make_backend(topology, params, workers=workers, gpu_device=gpu_device)


register_backend("gpu", kind="B200 persistent RK4 (sm_100a)",
                 requires="libsto_b200.so and an sm_100 GPU", probe=_gpu_probe,
                 factory=_gpu_factory)
