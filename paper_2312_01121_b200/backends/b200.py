"""The registered "gpu" backend: B200 persistent-kernel RK4 (sm_100a).

Replaces the reference's `TorchBackend` (`backends/gpu.py:49-119`) behind
the same registry id and factory signature. Two entry points:

* `derivative(m, u, out)` -- the reference plugin contract
  (`backends/__init__.py:5-7, 48-50`), one fused K0 launch. numpy arrays
  pay an H2D/D2H per call exactly like `gpu.py:87-88,118`; CUDA torch
  tensors are used in place (no copies), which is what
  `time_derivative_eval` wants to time.
* `integrate_run(m0, series, dt, steps, stride)` -- the whole time loop in
  one persistent launch; `integrate()` prefers it whenever present.

Device selection follows `gpu.py:40-46`: explicit argument, then the
SPINOSC_GPU_DEVICE environment variable, then 0; "cuda:<i>" strings are
accepted. Any non-CUDA device raises `BackendUnavailableError`: there is no
CPU evaluation behind this backend.
"""

from __future__ import annotations

import os

import numpy as np

from .. import _native
from ..errors import BackendUnavailableError, ParameterError
from ..params import kernel_scalars

ENV_DEVICE = "SPINOSC_GPU_DEVICE"


def is_available(device=None) -> bool:
    try:
        return _native.probe(resolve_device(device))
    except BackendUnavailableError:
        return False


def resolve_device(device=None) -> int:
    """Device ordinal from argument / env var / default 0 (ref `gpu.py:40-46`)."""
    if device is None:
        device = os.environ.get(ENV_DEVICE, 0)
    if isinstance(device, str) and device.startswith("cuda"):
        device = device.split(":", 1)[1] if ":" in device else 0
    try:
        return int(device)
    except (TypeError, ValueError):
        from . import available_backend_ids

        raise BackendUnavailableError("gpu", available_backend_ids()) from None


class B200Backend:
    """Coupled-STO equation of motion and RK4 time loop on one B200."""

    backend_id = "gpu"
    kind = "B200 persistent RK4 (sm_100a)"

    def __init__(self, topology, params, device=None, flags: int = 0, consts=None):
        """`consts` overrides the 11 kernel scalars derived from `params`;
        `flags` forces a kernel family (_native.FORCE_*; testing/benchmarks)."""
        self.device_index = resolve_device(device)
        if not _native.probe(self.device_index):
            from . import available_backend_ids

            raise BackendUnavailableError("gpu", available_backend_ids())
        import torch

        self._torch = torch
        self._dev = torch.device("cuda", self.device_index)
        self.n, self.n_in = topology.n, topology.n_in
        w = getattr(topology.coupling, "tensor", None)  # device-built W: used in place
        self._plan = _native.Plan(w if w is not None else topology.coupling.entries,
                                  topology.input_weights.entries,
                                  kernel_scalars(params) if consts is None else consts,
                                  device=self.device_index, flags=flags)
        self.last_kernel_seconds = float("nan")
        self._stage = None  # derivative(): page-locked / device staging, made on first use

    @property
    def device(self) -> str:
        return str(self._dev)

    @property
    def plan_info(self) -> dict:
        return dict(self._plan.info)

    def close(self) -> None:
        self._plan.close()

    # ------------------------------------------------------------------
    def derivative(self, m, u, out):
        """Write dm/dt at (m, u) into `out` (numpy or CUDA torch tensors)."""
        t = self._torch
        if isinstance(m, t.Tensor) and m.is_cuda:
            for a, shape in ((m, (self.n, 3)), (u, (self.n_in,)), (out, (self.n, 3))):
                if not (isinstance(a, t.Tensor) and a.is_cuda and tuple(a.shape) == shape and
                        a.dtype == t.float64 and a.is_contiguous() and
                        a.device.index == self.device_index):
                    raise ParameterError("derivative expects contiguous float64 CUDA tensors "
                                         f"m (n, 3), u (n_in,), out (n, 3) on {self._dev}")
            self._plan.derivative_dev(m, u, out)
            return out
        m = np.asarray(m, dtype=np.float64)
        u = np.asarray(u, dtype=np.float64)
        if m.shape != (self.n, 3) or u.shape != (self.n_in,):
            raise ParameterError("derivative expects m (n, 3) and u (n_in,)")
        # host buffers (the reference plugin contract, called once per RK stage
        # by derivative-only drivers): page-locked staging owned by the backend,
        # one H2D, the K0 launch, one D2H, one stream sync -- no per-call
        # allocation or pageable copies
        st = self._stage
        if st is None:
            k = 3 * self.n + self.n_in
            st = self._stage = (t.empty(k, dtype=t.float64, pin_memory=True),
                                t.empty(k, dtype=t.float64, device=self._dev),
                                t.empty(3 * self.n, dtype=t.float64, device=self._dev),
                                t.empty(3 * self.n, dtype=t.float64, pin_memory=True))
        h_in, d_in, d_out, h_out = st
        hv = h_in.numpy()
        hv[:3 * self.n] = m.reshape(-1)
        hv[3 * self.n:] = u
        with t.cuda.device(self._dev):
            d_in.copy_(h_in, non_blocking=True)
            self._plan.derivative_dev(d_in[:3 * self.n].view(self.n, 3), d_in[3 * self.n:],
                                      d_out.view(self.n, 3))
            h_out.copy_(d_out, non_blocking=True)
            t.cuda.current_stream(self._dev).synchronize()
        np.copyto(out, h_out.numpy().reshape(self.n, 3))
        return out

    def integrate_run(self, m0: np.ndarray, samples: np.ndarray, steps_per_sample: int,
                      dt: float, steps: int, stride: int) -> np.ndarray:
        """Run the whole RK4 loop on the device; returns the recorded states.

        m0 is updated in place to the final state. Raises
        IntegrationDivergedError(oscillator, step) like `integrator.py:174-177`.
        """
        t = self._torch
        samples = np.asarray(samples, dtype=np.float64)
        if np.shape(m0) != (self.n, 3):
            raise ParameterError(f"m0 must be ({self.n}, 3), got {np.shape(m0)}")
        if samples.ndim != 2 or samples.shape[1] != self.n_in or samples.shape[0] < 1:
            raise ParameterError(f"drive samples must be (n_samples, {self.n_in}), "
                                 f"got {samples.shape}")
        nrec = _native.n_records(steps, stride)
        with t.cuda.device(self._dev):
            m_d = t.as_tensor(np.ascontiguousarray(m0, dtype=np.float64)).to(self._dev)
            s_d = t.as_tensor(np.ascontiguousarray(samples, dtype=np.float64)).to(self._dev)
            states_d = t.empty((nrec, self.n, 3), dtype=t.float64, device=self._dev)
            start, stop = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
            start.record()
            self._plan.integrate_dev(m_d, s_d, steps_per_sample, dt, steps, stride, states_d,
                                     sync=False)
            stop.record()
            stop.synchronize()
            self.last_kernel_seconds = start.elapsed_time(stop) / 1e3
            self._plan.last_status()  # raises IntegrationDivergedError on divergence
            # Trajectory.max_norm_drift on the device (bit-identical to the host
            # numpy pass, which costs more than a densely recorded run itself)
            drift_d = _native.norm_drift(states_d)
            states = _to_host(t, states_d)
            self.last_norm_drift = float(drift_d.item())
            np.copyto(m0, m_d.cpu().numpy())
        return states


    def integrate_ensemble_run(self, consts: np.ndarray, samples: np.ndarray,
                               steps_per_sample: int, dt: float, steps: int, stride: int,
                               m0: np.ndarray, exact: bool = False) -> np.ndarray:
        """B members sharing W/W_in: consts (B, 11), m0 (B, n, 3) updated in place,
        samples (n_samples, n_in) shared or (B, n_samples, n_in) per member.
        Returns states (n_records, B, n, 3).  exact=True: bit-exact CUDA-core
        path (each member == integrate() with its parameters) instead of DMMA."""
        t = self._torch
        consts = np.ascontiguousarray(consts, dtype=np.float64)
        batch = consts.shape[0]
        if consts.shape != (batch, 11) or m0.shape != (batch, self.n, 3):
            raise ParameterError("ensemble expects consts (B, 11) and m0 (B, n, 3)")
        samples = np.ascontiguousarray(samples, dtype=np.float64)
        per_member = samples.ndim == 3
        if per_member and samples.shape[0] != batch:
            raise ParameterError("per-member drive must be (B, n_samples, n_in)")
        if samples.ndim not in (2, 3) or samples.shape[-1] != self.n_in or samples.shape[-2] < 1:
            raise ParameterError(f"drive samples must be ([B,] n_samples, {self.n_in})")
        stride_m = samples.shape[1] * samples.shape[2] if per_member else 0
        nrec = _native.n_records(steps, stride)
        with t.cuda.device(self._dev):
            c_d = t.as_tensor(consts).to(self._dev)
            m_d = t.as_tensor(np.ascontiguousarray(m0, dtype=np.float64)).to(self._dev)
            s_d = t.as_tensor(samples).to(self._dev)
            states_d = t.empty((nrec, batch, self.n, 3), dtype=t.float64, device=self._dev)
            start, stop = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
            start.record()
            self._plan.integrate_ensemble_dev(m_d, c_d, s_d, steps_per_sample, stride_m, dt,
                                              steps, stride, states_d, exact=exact)
            stop.record()
            stop.synchronize()
            self.last_kernel_seconds = start.elapsed_time(stop) / 1e3
            drift_d = _native.norm_drift(states_d, members=batch)
            states = _to_host(t, states_d)
            self.last_norm_drift_members = drift_d.cpu().numpy()
            np.copyto(m0, m_d.cpu().numpy())
        return states


def _to_host(t, tensor):
    """Device -> host through page-locked memory (torch's caching host allocator
    reuses the block once the previous result is released): one DMA at full
    PCIe rate instead of a pageable staging copy."""
    host = t.empty(tensor.shape, dtype=tensor.dtype, pin_memory=True)
    host.copy_(tensor)
    return host.numpy()


def make_backend(topology, params, workers=None, gpu_device=None):
    """Registry factory, signature of ref `backends/__init__.py:48-50`."""
    return B200Backend(topology, params, device=gpu_device)
