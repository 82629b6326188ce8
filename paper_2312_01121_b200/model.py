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


def llg_derivative(m, u, topology, params, consts=None, out=None, workspace=None):
    """dm/dt for the whole array, evaluated by the K0 kernel on the GPU.

    Same contract as ref `model.py:206-302`: writes only `out` (allocated when
    None). `consts` and `workspace` are accepted for signature compatibility;
    the device plan owns its scratch.
    """
    from .backends.b200 import B200Backend

    m = np.ascontiguousarray(np.asarray(m, dtype=np.float64))
    if out is None:
        out = np.empty_like(m)
    B200Backend(topology, params).derivative(m, np.asarray(u, dtype=np.float64), out)
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
