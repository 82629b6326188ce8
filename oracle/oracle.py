"""ctypes front end of the CPU parity oracle (TEST INFRASTRUCTURE ONLY).

Loaded by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` leg -- never by the product package. Wraps
oracle/libsto_oracle.so (sto_oracle.c, a strict-IEEE restatement of the
reference's `_row_derivative`/`_tree_reduce`/`rk4_step`/`integrate`).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "libsto_oracle.so"

_P = ctypes.POINTER(ctypes.c_double)
_I64P = ctypes.POINTER(ctypes.c_int64)
_lib = None


def build(force: bool = False) -> Path:
    """Compile libsto_oracle.so with the committed Makefile (strict IEEE flags)."""
    src = HERE / "sto_oracle.c"
    if force or not LIB_PATH.exists() or LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-C", str(HERE), "-s"], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(LIB_PATH))
        L.sto_oracle_tree_sum.restype = ctypes.c_double
        L.sto_oracle_tree_sum.argtypes = [_P, ctypes.c_int64]
        L.sto_oracle_derivative.restype = ctypes.c_int
        L.sto_oracle_derivative.argtypes = [ctypes.c_int64, ctypes.c_int64, _P, _P, _P,
                                            _P, _P, _P, ctypes.c_int]
        L.sto_oracle_integrate.restype = ctypes.c_int
        L.sto_oracle_integrate.argtypes = [
            ctypes.c_int64, ctypes.c_int64, _P, _P, _P, _P, _P, ctypes.c_int64,
            ctypes.c_int64, ctypes.c_double, ctypes.c_int64, ctypes.c_int64, _P,
            _I64P, _I64P, ctypes.c_int]
        L.sto_oracle_n_records.restype = ctypes.c_int64
        L.sto_oracle_n_records.argtypes = [ctypes.c_int64, ctypes.c_int64]
        L.sto_oracle_max_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_P)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def default_threads() -> int:
    return int(os.environ.get("STO_ORACLE_THREADS", os.cpu_count() or 1))


def tree_sum(values) -> float:
    buf = _f64(values).copy()
    return float(lib().sto_oracle_tree_sum(_ptr(buf), buf.size))


def derivative(w_cp, w_in, consts, m, u, threads: int = 1) -> np.ndarray:
    w_cp, w_in, m, u = _f64(w_cp), _f64(w_in), _f64(m), _f64(u)
    c = _f64(consts)
    out = np.empty_like(m)
    rc = lib().sto_oracle_derivative(w_cp.shape[0], w_in.shape[1], _ptr(w_cp), _ptr(w_in),
                                     _ptr(c), _ptr(m), _ptr(u), _ptr(out), threads)
    if rc:
        raise RuntimeError(f"oracle derivative failed rc={rc}")
    return out


class OracleDiverged(RuntimeError):
    def __init__(self, oscillator: int, step: int):
        super().__init__(f"oracle diverged at oscillator {oscillator}, step {step}")
        self.oscillator, self.step = oscillator, step


def integrate(w_cp, w_in, consts, m0, samples, steps_per_sample, dt, steps, stride,
              threads: int | None = None):
    """Returns (states (R, n, 3), final m). Raises OracleDiverged like the reference."""
    w_cp, w_in, samples = _f64(w_cp), _f64(w_in), _f64(samples)
    c = _f64(consts)
    m = _f64(m0).copy()
    n, n_in = w_cp.shape[0], w_in.shape[1]
    n_rec = lib().sto_oracle_n_records(steps, stride)
    states = np.empty((n_rec, n, 3))
    bad_osc, bad_step = ctypes.c_int64(-1), ctypes.c_int64(-1)
    rc = lib().sto_oracle_integrate(
        n, n_in, _ptr(w_cp), _ptr(w_in), _ptr(c), _ptr(m), _ptr(samples),
        samples.shape[0], steps_per_sample, float(dt), steps, stride, _ptr(states),
        ctypes.byref(bad_osc), ctypes.byref(bad_step),
        default_threads() if threads is None else threads)
    if rc == 3:
        raise OracleDiverged(bad_osc.value, bad_step.value)
    if rc:
        raise RuntimeError(f"oracle integrate failed rc={rc}")
    return states, m
