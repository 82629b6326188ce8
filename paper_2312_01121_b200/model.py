"""Drive series (zero-order hold) and GPU-evaluated model functions.

`InputSeries` mirrors `spinosc/model.py:93-149`: sample s is held for steps
[s*sps, (s+1)*sps) and all four RK stages of a step see the same sample;
a one-sample series is constant for any run length.

`llg_derivative`, `tree_matvec` and `tree_reduce_rows` keep the reference
names (`model.py:31-63, 206-302`) but evaluate on the B200 through the
C-ABI (`sto_derivative`, `sto_tree_matvec`); there is no CPU evaluation in
this package. Their results are bit-identical to the reference's pinned
operation order.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ParameterError


@dataclass(frozen=True)
class InputSeries:
    """(n_samples, n_in) float64 drive samples held for `steps_per_sample` steps."""

    samples: np.ndarray
    steps_per_sample: int = 1

    def __post_init__(self) -> None:
        s = np.ascontiguousarray(np.asarray(self.samples, dtype=np.float64))
        if s.ndim != 2 or s.shape[0] < 1 or s.shape[1] < 1:
            raise ParameterError("input samples must be a (n_samples, n_in) array")
        if not np.isfinite(s).all():
            raise ParameterError("input samples must be finite")
        if self.steps_per_sample < 1:
            raise ParameterError("steps_per_sample must be >= 1")
        object.__setattr__(self, "samples", s)

    @classmethod
    def zeros(cls, n_in: int) -> "InputSeries":
        return cls(samples=np.zeros((1, n_in)), steps_per_sample=1)

    @property
    def n_in(self) -> int:
        return self.samples.shape[1]

    @property
    def n_samples(self) -> int:
        return self.samples.shape[0]

    def check_steps(self, steps: int) -> None:
        """A multi-sample series must cover exactly the samples a run consumes."""
        if self.n_samples == 1:
            return
        lo = (self.n_samples - 1) * self.steps_per_sample
        hi = self.n_samples * self.steps_per_sample
        if not lo < steps <= hi:
            raise ParameterError(
                f"input series with {self.n_samples} samples held for "
                f"{self.steps_per_sample} steps covers ({lo}, {hi}] steps, got {steps}"
            )

    def sample_for_step(self, step: int) -> np.ndarray:
        """Sample active during 0-based `step` (a view, no copy)."""
        if self.n_samples == 1:
            return self.samples[0]
        return self.samples[step // self.steps_per_sample]


class Workspace:
    """Shape tag of the reference's `Workspace` (`model.py:66-90`).

    The reference preallocates host scratch (an n*n product buffer among it)
    for its numpy derivative; here the device plan owns all scratch, so this
    only records (n, n_in) for code that constructs and passes one around.
    """

    def __init__(self, n: int, n_in: int):
        self.n = int(n)
        self.n_in = int(n_in)


def effective_field(m, params, consts=None) -> np.ndarray:
    """(0, 0, h_appl + h_aniso m_z) per oscillator (ref `model.py:152-161`)."""
    from .params import derive

    consts = derive(params) if consts is None else consts
    m = np.asarray(m, dtype=np.float64)
    out = np.zeros_like(m)
    out[:, 2] = params.h_appl + consts.h_aniso * m[:, 2]
    return out


def spin_torque_strength(m, params, consts=None) -> np.ndarray:
    """h_s(m) = prefactor / (1 + lambda m.p), in Oe (ref `model.py:164-173`)."""
    from .params import derive

    consts = derive(params) if consts is None else consts
    m = np.asarray(m, dtype=np.float64)
    mdotp = m[:, 0] * consts.px + m[:, 1] * consts.py + m[:, 2] * consts.pz
    return consts.h_s_prefactor / (1.0 + params.lambda_stt * mdotp)


_MATVEC_PLANS: dict = {}  # id(coupling) -> (weakref(coupling), Plan)


def _matvec_plan_for(coupling):
    """One device plan (W layout resident) per CouplingMatrix object, reused by
    every coupling_field_x call on it; dies with the object."""
    import weakref

    from . import _native

    key = id(coupling)
    hit = _MATVEC_PLANS.get(key)
    if hit is None or hit[0]() is not coupling:
        import os

        n = coupling.n
        if hasattr(coupling, "tensor"):  # DeviceCouplingMatrix: W already on its GPU
            w, device = coupling.tensor, coupling.tensor.device.index
        else:
            w, device = coupling.entries, int(os.environ.get("SPINOSC_GPU_DEVICE", 0))
        plan = _native.Plan(w, np.zeros((n, 1)), [0.0] * 11, device=device)
        hit = (weakref.ref(coupling, lambda _r, k=key: _MATVEC_PLANS.pop(k, None)), plan)
        _MATVEC_PLANS[key] = hit
    return hit[1]


def coupling_field_x(coupling, m_x, a_cp: float) -> np.ndarray:
    """a_cp (W_cp m^x) with the pinned tree on the GPU (ref `model.py:176-180`).

    For a CouplingMatrix the device plan (W uploaded and laid out once) is cached
    on the object, so a call costs the m^x upload and one matvec launch
    (`sto_plan_matvec`); a raw array goes through the one-shot `tree_matvec`."""
    m_x = np.asarray(m_x, dtype=np.float64)
    if hasattr(coupling, "entries") and hasattr(coupling, "n"):
        import torch

        plan = _matvec_plan_for(coupling)
        dev = torch.device("cuda", plan.device)
        x = torch.as_tensor(np.ascontiguousarray(m_x)).to(dev)
        out = torch.empty(coupling.n, dtype=torch.float64, device=dev)
        plan.matvec_dev(x, out)
        return a_cp * out.cpu().numpy()
    return a_cp * tree_matvec(np.asarray(coupling, dtype=np.float64), m_x)


def input_field_x(weights, u, a_in: float) -> np.ndarray:
    """a_in (W_in u) with the pinned tree on the GPU (ref `model.py:183-187`)."""
    entries = getattr(weights, "entries", weights)
    return a_in * tree_matvec(np.asarray(entries, dtype=np.float64), np.asarray(u, dtype=np.float64))


def total_b(m, u, topology, params, consts=None) -> np.ndarray:
    """Full local field b_k, shape (n, 3), same operation order as ref `model.py:190-203`."""
    from .params import derive

    consts = derive(params) if consts is None else consts
    m = np.asarray(m, dtype=np.float64)
    mx, my, mz = m[:, 0], m[:, 1], m[:, 2]
    hs = spin_torque_strength(m, params, consts)
    cpx = coupling_field_x(topology.coupling, mx, params.a_cp)
    inx = input_field_x(topology.input_weights, np.asarray(u, dtype=np.float64), params.a_in)
    px, py, pz = consts.px, consts.py, consts.pz
    b = np.empty_like(m)
    b[:, 0] = (cpx + inx) + hs * (py * mz - pz * my)
    b[:, 1] = hs * (pz * mx - px * mz)
    b[:, 2] = (params.h_appl + consts.h_aniso * mz) + hs * (px * my - py * mx)
    return b


_BACKENDS: dict = {}  # id(topology) -> (weakref(topology), {scalars: B200Backend})


def _backend_for(topology, scalars: tuple):
    """One B200 plan per (topology, kernel scalars), reused across calls: the W
    upload and layout permute happen once, like the reference's TorchBackend
    copying W at construction (gpu.py:68-71).  Entries die with the topology."""
    import weakref

    from .backends.b200 import B200Backend

    key = id(topology)
    hit = _BACKENDS.get(key)
    if hit is None or hit[0]() is not topology:
        hit = (weakref.ref(topology, lambda _r, k=key: _BACKENDS.pop(k, None)), {})
        _BACKENDS[key] = hit
    plans = hit[1]
    if scalars not in plans:
        if len(plans) >= 4:  # a parameter sweep through this helper: keep the newest few
            plans.pop(next(iter(plans))).close()
        plans[scalars] = B200Backend(topology, None, consts=scalars)
    return plans[scalars]


def llg_derivative(m, u, topology, params, consts=None, out=None, workspace=None):
    """dm/dt for the whole array, evaluated by the K0 kernel on the GPU.

    Same contract as ref `model.py:206-302`: writes only `out` (allocated when
    None); `consts` (a DerivedConstants) replaces `derive(params)` as in the
    reference.  The device plan for (topology, scalars) is cached, so repeated
    calls pay only the m/u/out copies.  `workspace` is accepted for signature
    compatibility; the device plan owns its scratch.
    """
    from .params import kernel_scalars

    m = np.ascontiguousarray(np.asarray(m, dtype=np.float64))
    if out is None:
        out = np.empty_like(m)
    backend = _backend_for(topology, tuple(float(v) for v in kernel_scalars(params, consts)))
    backend.derivative(m, np.asarray(u, dtype=np.float64), out)
    return out


def tree_matvec(matrix, vec, out=None):
    """(matrix @ vec) summed with the pinned adjacent-pairs tree, on the GPU."""
    from . import _native

    return _native.tree_matvec(matrix, vec, out)


def tree_reduce_rows(products, halvebuf=None, out=None):
    """Row sums of `products` with the pinned tree (ref `model.py:31-52`), on the GPU.

    `halvebuf` is accepted for signature compatibility and left untouched.
    """
    from . import _native

    products = np.asarray(products, dtype=np.float64)
    ones = np.ones(products.shape[1])
    return _native.tree_matvec(products, ones, out)
