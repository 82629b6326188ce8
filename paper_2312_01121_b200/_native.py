"""ctypes binding of libsto_b200.so (the C ABI in include/sto.h).

There is no fallback: if the library is missing or no sm_100 device is
present, every entry point raises (`BackendUnavailableError` for the probe
path, `SpinoscError` otherwise). Device buffers are torch tensors; only raw
pointers and sizes cross the ABI.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

from .errors import (BackendUnavailableError, IntegrationDivergedError, ParameterError,
                     SpinoscError)

# STO_LIB: load another build of the same ABI from this directory (A/B timing of variants)
LIB_PATH = Path(__file__).resolve().parent / os.environ.get("STO_LIB", "libsto_b200.so")

STO_OK, STO_E_UNAVAILABLE, STO_E_PARAM, STO_E_DIVERGED, STO_E_CUDA, STO_E_NOMEM = range(6)

# flags of sto_plan_desc (include/sto.h)
FORCE_STREAM, FORCE_RESIDENT, FORCE_SINGLE, NO_TINY, FORCE_REG, NO_REG = (
    0x1, 0x2, 0x4, 0x8, 0x10, 0x20)
FORCE_CLUSTER, NO_CLUSTER = 0x40, 0x80
KERNEL_NAMES = {0: "tiny", 1: "single", 2: "resident", 3: "stream", 4: "reg", 5: "cluster"}

_c_double_p = ctypes.POINTER(ctypes.c_double)


class PlanDesc(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("n_in", ctypes.c_int64),
                ("w_cp", ctypes.c_void_p), ("ld_cp", ctypes.c_int64),
                ("w_in", ctypes.c_void_p), ("ld_in", ctypes.c_int64),
                ("consts", ctypes.c_double * 11), ("device", ctypes.c_int),
                ("flags", ctypes.c_int), ("row_begin", ctypes.c_int64),
                ("row_count", ctypes.c_int64), ("world", ctypes.c_int32),
                ("rank", ctypes.c_int32)]


class Run(ctypes.Structure):
    _fields_ = [("m", ctypes.c_void_p), ("samples", ctypes.c_void_p),
                ("n_samples", ctypes.c_int64), ("steps_per_sample", ctypes.c_int64),
                ("dt", ctypes.c_double), ("steps", ctypes.c_int64),
                ("record_stride", ctypes.c_int64), ("states", ctypes.c_void_p)]


class Status(ctypes.Structure):
    _fields_ = [("diverged", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("oscillator", ctypes.c_int64), ("step", ctypes.c_int64)]


class EnsembleRun(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int64), ("consts", ctypes.c_void_p), ("m", ctypes.c_void_p),
                ("samples", ctypes.c_void_p), ("n_samples", ctypes.c_int64),
                ("steps_per_sample", ctypes.c_int64), ("sample_member_stride", ctypes.c_int64),
                ("dt", ctypes.c_double), ("steps", ctypes.c_int64),
                ("record_stride", ctypes.c_int64), ("states", ctypes.c_void_p)]


class PlanInfo(ctypes.Structure):
    _fields_ = [("kernel", ctypes.c_int32), ("grid", ctypes.c_int32),
                ("threads", ctypes.c_int32), ("smem_bytes", ctypes.c_int32),
                ("ldw", ctypes.c_int64), ("block_cols", ctypes.c_int64),
                ("w_bytes", ctypes.c_int64), ("x_window_cols", ctypes.c_int64)]


# every symbol include/sto.h declares, with its ctypes signature
SIGNATURES = {
    "sto_last_error": (ctypes.c_char_p, []),
    "sto_abi_version": (ctypes.c_int, []),
    "sto_probe": (ctypes.c_int, [ctypes.c_int]),
    "sto_n_records": (ctypes.c_int64, [ctypes.c_int64, ctypes.c_int64]),
    "sto_plan_create": (ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(PlanDesc)]),
    "sto_plan_destroy": (None, [ctypes.c_void_p]),
    "sto_plan_get_info": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(PlanInfo)]),
    "sto_derivative": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                      ctypes.c_void_p, ctypes.c_void_p]),
    "sto_integrate": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(Run),
                                     ctypes.POINTER(Status), ctypes.c_void_p]),
    "sto_integrate_ensemble": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(EnsembleRun),
                                              ctypes.POINTER(Status), ctypes.c_void_p]),
    "sto_plan_last_status": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(Status),
                                            ctypes.c_void_p]),
    "sto_integrate_ensemble_exact": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(EnsembleRun),
                                                    ctypes.POINTER(Status), ctypes.c_void_p]),
    "sto_plan_exchange_handle": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p,
                                                ctypes.c_int64]),
    "sto_plan_connect": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32]),
    "sto_plan_connect_local": (ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int32]),
    "sto_integrate_group": (ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int32,
                                           ctypes.POINTER(Run), ctypes.POINTER(Status),
                                           ctypes.c_void_p]),
    "sto_integrate_host": (ctypes.c_int, [ctypes.c_void_p, _c_double_p, _c_double_p,
                                          ctypes.c_int64, ctypes.c_int64, ctypes.c_double,
                                          ctypes.c_int64, ctypes.c_int64, _c_double_p,
                                          ctypes.POINTER(Status)]),
    "sto_tree_matvec": (ctypes.c_int, [ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                                       _c_double_p, ctypes.c_int64, _c_double_p, _c_double_p]),
    "sto_pcg64_fill": (ctypes.c_int, [ctypes.c_int, ctypes.c_void_p, ctypes.c_int64,
                                      ctypes.c_int64, ctypes.POINTER(ctypes.c_uint64),
                                      ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p]),
    "sto_gemv": (ctypes.c_int, [ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "sto_scale_div": (ctypes.c_int, [ctypes.c_int, ctypes.c_void_p, ctypes.c_int64,
                                     ctypes.c_double, ctypes.c_void_p]),
    "sto_norm_drift": (ctypes.c_int, [ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                      ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]),
    "sto_plan_matvec": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_void_p]),
    "sto_selftest_div": (ctypes.c_int, [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_void_p]),
    "sto_write_trajectory_csv": (ctypes.c_int, [ctypes.c_char_p, _c_double_p, _c_double_p,
                                                ctypes.c_int64, ctypes.c_int64, ctypes.c_int32]),
}

_lib = None


def lib():
    """Load libsto_b200.so once; raise loudly when it is absent."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise SpinoscError(
                f"{LIB_PATH.name} is not built; run `python -c 'import __graft_entry__ as g; "
                f"g.build()'` (or `make -C paper_2312_01121_b200/csrc`)")
        L = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            if "STO_LIB" in os.environ and not hasattr(L, name):
                continue  # an older A/B variant build: entry points added since are absent
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def last_error() -> str:
    return lib().sto_last_error().decode(errors="replace")


def check(rc: int, status: Status | None = None) -> None:
    if rc == STO_OK:
        return
    msg = last_error()
    if rc == STO_E_DIVERGED and status is not None:
        raise IntegrationDivergedError(oscillator=status.oscillator, step=status.step)
    if rc == STO_E_PARAM:
        raise ParameterError(msg)
    if rc == STO_E_UNAVAILABLE:
        raise BackendUnavailableError("gpu", [])
    raise SpinoscError(f"sto error {rc}: {msg}")


def probe(device: int = 0) -> bool:
    """True when the library loads and `device` is an sm_100 GPU (never raises)."""
    try:
        return bool(lib().sto_probe(int(device)))
    except Exception:
        return False


def n_records(steps: int, stride: int) -> int:
    return int(lib().sto_n_records(steps, stride))


def _torch():
    import torch

    return torch


def _stream_ptr(device: int):
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def pcg64_words(seed: int) -> tuple[int, int, int, int]:
    """(state_hi, state_lo, inc_hi, inc_lo) of numpy's PCG64(seed) before any draw."""
    st = np.random.PCG64(seed).state["state"]
    m64 = (1 << 64) - 1
    return (st["state"] >> 64, st["state"] & m64, st["inc"] >> 64, st["inc"] & m64)


def pcg64_fill(out, count: int, offset: int, words, diag_n: int = 0, ld: int = 0) -> None:
    """Device draws of RngStream.uniform_pm1 (sto_pcg64_fill); `out` a CUDA float64 tensor."""
    w = (ctypes.c_uint64 * 4)(*[int(v) for v in words])
    dev = out.device.index
    check(lib().sto_pcg64_fill(dev, out.data_ptr(), int(count), int(offset), w, int(diag_n),
                               int(ld), _stream_ptr(dev)))


def write_trajectory_csv(path, times: np.ndarray, states: np.ndarray, threads: int = 0) -> None:
    """Native parallel `t,k,mx,my,mz` writer (sto_write_trajectory_csv)."""
    t = np.ascontiguousarray(times, dtype=np.float64)
    s = np.ascontiguousarray(states, dtype=np.float64)
    if s.ndim != 3 or s.shape[2] != 3 or t.shape != (s.shape[0],):
        raise ParameterError("write_trajectory_csv expects times (R,) and states (R, n, 3)")
    rc = lib().sto_write_trajectory_csv(os.fsencode(path), t.ctypes.data_as(_c_double_p),
                                        s.ctypes.data_as(_c_double_p), s.shape[0], s.shape[1],
                                        int(threads))
    if rc != STO_OK:
        raise ParameterError(f"cannot write trajectory CSV to {path!s}")


def gemv(w, x, y) -> None:
    """y = w @ x on the device (unpinned order; spectral-radius matvecs)."""
    dev = w.device.index
    check(lib().sto_gemv(dev, w.data_ptr(), w.shape[0], w.shape[1], w.stride(0), x.data_ptr(),
                         y.data_ptr(), _stream_ptr(dev)))


def scale_div(a, divisor: float) -> None:
    """a /= divisor in place (IEEE division) on the device."""
    dev = a.device.index
    check(lib().sto_scale_div(dev, a.data_ptr(), a.numel(), float(divisor), _stream_ptr(dev)))


def norm_drift(states, members: int = 1):
    """max | |m| - 1 | per member of device states (outer, members, n, 3) -> CUDA
    tensor (members,); Trajectory.max_norm_drift on the device."""
    import torch

    dev = states.device.index
    out = torch.empty((members,), dtype=torch.float64, device=states.device)
    outer = states.numel() // (3 * members * states.shape[-2]) if states.numel() else 0
    check(lib().sto_norm_drift(dev, states.data_ptr(), outer, members, states.shape[-2],
                               out.data_ptr(), _stream_ptr(dev)))
    return out


def selftest_div(a, b):
    """(q, ok, ref) of the kernels' speculative division vs __ddiv_rn (test hook)."""
    import torch

    dev = a.device.index
    q = torch.empty_like(a)
    ref = torch.empty_like(a)
    ok = torch.empty(a.shape, dtype=torch.int32, device=a.device)
    check(lib().sto_selftest_div(dev, a.data_ptr(), b.data_ptr(), a.numel(), q.data_ptr(),
                                 ok.data_ptr(), ref.data_ptr(), _stream_ptr(dev)))
    return q, ok, ref


class Plan:
    """Owns a device-resident W layout + launch configuration (sto_plan)."""

    def __init__(self, w_cp, w_in: np.ndarray, consts, device: int = 0,
                 flags: int = 0, shard: tuple[int, int, int, int] | None = None):
        """shard = (row_begin, row_count, world, rank): w_cp / w_in hold only the
        shard's rows (row_count x n and row_count x n_in).  w_cp may be a host
        array or a CUDA float64 tensor (device-built W: no host round trip)."""
        if hasattr(w_cp, "data_ptr") and getattr(w_cp, "is_cuda", False):
            w_cp = w_cp.contiguous()  # device-resident W (keeps the tensor alive below)
            if w_cp.dtype != _torch().float64 or w_cp.device.index != int(device):
                raise ParameterError("device coupling must be float64 on the plan's device")
            w_ptr, shape = w_cp.data_ptr(), tuple(w_cp.shape)
        else:
            w_cp = np.ascontiguousarray(w_cp, dtype=np.float64)
            w_ptr, shape = w_cp.ctypes.data, w_cp.shape
        w_in = np.ascontiguousarray(w_in, dtype=np.float64)
        if len(shape) != 2:
            raise ParameterError("coupling matrix must be square")
        rows, n = shape
        if shard is None and rows != n:
            raise ParameterError("coupling matrix must be square")
        if w_in.ndim != 2 or w_in.shape[0] != rows:
            raise ParameterError("input weights must be (n, n_in)")
        self.n, self.n_in = n, w_in.shape[1]
        self.device = int(device)
        self.shard = shard
        d = PlanDesc(n=self.n, n_in=self.n_in, w_cp=w_ptr, ld_cp=self.n,
                     w_in=w_in.ctypes.data, ld_in=self.n_in, device=self.device, flags=flags)
        if shard is not None:
            d.row_begin, d.row_count, d.world, d.rank = (int(v) for v in shard)
            if d.row_count != rows:
                raise ParameterError("shard row_count must equal the rows passed")
        for i, v in enumerate(consts):
            d.consts[i] = float(v)
        h = ctypes.c_void_p()
        check(lib().sto_plan_create(ctypes.byref(h), ctypes.byref(d)))
        self._h = h
        info = PlanInfo()
        check(lib().sto_plan_get_info(self._h, ctypes.byref(info)))
        self.info = {k: getattr(info, k) for k, _ in PlanInfo._fields_}
        self.info["kernel_name"] = KERNEL_NAMES.get(info.kernel, "?")

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().sto_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- device-pointer entry points (torch CUDA tensors) -----------------
    def derivative_dev(self, m, u, out) -> None:
        check(lib().sto_derivative(self._h, m.data_ptr(), u.data_ptr(), out.data_ptr(),
                                   _stream_ptr(self.device)))

    def integrate_dev(self, m, samples, steps_per_sample: int, dt: float, steps: int,
                      stride: int, states, sync: bool = True) -> Status:
        run = Run(m=m.data_ptr(), samples=samples.data_ptr(), n_samples=samples.shape[0],
                  steps_per_sample=int(steps_per_sample), dt=float(dt), steps=int(steps),
                  record_stride=int(stride),
                  states=states.data_ptr() if states is not None else None)
        st = Status()
        rc = lib().sto_integrate(self._h, ctypes.byref(run),
                                 ctypes.byref(st) if sync else None, _stream_ptr(self.device))
        check(rc, st)
        return st

    def matvec_dev(self, x, out) -> None:
        """out = pinned-tree W @ x with the plan's resident W (device tensors)."""
        check(lib().sto_plan_matvec(self._h, x.data_ptr(), out.data_ptr(), _stream_ptr(self.device)))

    def integrate_ensemble_dev(self, m, consts, samples, steps_per_sample: int,
                               sample_member_stride: int, dt: float, steps: int, stride: int,
                               states, exact: bool = False) -> Status:
        """Batched members (m: (B, n, 3), consts: (B, 11)); synchronous status.
        exact: the bit-exact CUDA-core path (sto_integrate_ensemble_exact) instead
        of the DMMA tensor-core path."""
        run = EnsembleRun(batch=m.shape[0], consts=consts.data_ptr(), m=m.data_ptr(),
                          samples=samples.data_ptr(), n_samples=samples.shape[-2],
                          steps_per_sample=int(steps_per_sample),
                          sample_member_stride=int(sample_member_stride), dt=float(dt),
                          steps=int(steps), record_stride=int(stride),
                          states=states.data_ptr() if states is not None else None)
        st = Status()
        fn = lib().sto_integrate_ensemble_exact if exact else lib().sto_integrate_ensemble
        rc = fn(self._h, ctypes.byref(run), ctypes.byref(st), _stream_ptr(self.device))
        if rc == STO_E_DIVERGED:
            from .errors import IntegrationDivergedError

            err = IntegrationDivergedError(oscillator=st.oscillator, step=st.step)
            err.member = st.reserved
            raise err
        check(rc, st)
        return st

    def exchange_handle(self) -> bytes:
        buf = ctypes.create_string_buffer(64)
        check(lib().sto_plan_exchange_handle(self._h, buf, 64))
        return buf.raw

    def connect(self, handles: list[bytes]) -> None:
        blob = b"".join(handles)
        check(lib().sto_plan_connect(self._h, blob, len(handles)))

    def last_status(self) -> Status:
        st = Status()
        check(lib().sto_plan_last_status(self._h, ctypes.byref(st), _stream_ptr(self.device)),
              st)
        return st


def tree_matvec(matrix, vec, out=None, device: int | None = None):
    """Pinned-tree (matrix @ vec) on the GPU (model.py:55-63 semantics)."""
    a = np.ascontiguousarray(np.asarray(matrix, dtype=np.float64))
    x = np.ascontiguousarray(np.asarray(vec, dtype=np.float64))
    if a.ndim != 2 or x.ndim != 1 or a.shape[1] != x.shape[0]:
        raise ParameterError("tree_matvec needs a (rows, cols) matrix and a (cols,) vector")
    res = np.empty(a.shape[0])
    if device is None:
        device = int(os.environ.get("SPINOSC_GPU_DEVICE", 0))
    check(lib().sto_tree_matvec(int(device), a.shape[0], a.shape[1],
                                a.ctypes.data_as(_c_double_p), a.shape[1],
                                x.ctypes.data_as(_c_double_p), res.ctypes.data_as(_c_double_p)))
    if out is None:
        return res
    np.copyto(out, res)
    return out


def connect_local(plans: list["Plan"]) -> None:
    arr = (ctypes.c_void_p * len(plans))(*[p._h.value for p in plans])
    check(lib().sto_plan_connect_local(arr, len(plans)))


def integrate_group(plans: list["Plan"], m, samples, steps_per_sample: int, dt: float,
                    steps: int, stride: int, states) -> Status:
    """Logical ranks of one device in one persistent launch (synchronous)."""
    arr = (ctypes.c_void_p * len(plans))(*[p._h.value for p in plans])
    run = Run(m=m.data_ptr(), samples=samples.data_ptr(), n_samples=samples.shape[0],
              steps_per_sample=int(steps_per_sample), dt=float(dt), steps=int(steps),
              record_stride=int(stride), states=states.data_ptr() if states is not None else None)
    st = Status()
    rc = lib().sto_integrate_group(arr, len(plans), ctypes.byref(run), ctypes.byref(st),
                                   _stream_ptr(plans[0].device))
    check(rc, st)
    return st
