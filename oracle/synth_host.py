"""TEST / BASELINE INFRASTRUCTURE: host float64 generation of the synthetic
expert weights (the twin of csrc/synth.cu and paper_2511_10054_b200/synth.py)
through oracle/c/synth_host.c, threaded from Python (ctypes drops the GIL).
Used by bench.py's CPU reference arm; falls back to the numpy twin when the
C helper is not built (`make -C oracle`)."""

from __future__ import annotations

import ctypes as C
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libsynth_host.so")
_h = None


def _lib():
    global _h
    if _h is None and os.path.exists(_LIB):
        _h = C.CDLL(_LIB)
        _h.synth_f64_range.restype = None
        _h.synth_f64_range.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]
        _h.synth_mix_f64_range.restype = None
        _h.synth_mix_f64_range.argtypes = [C.c_uint64, C.c_uint64, C.c_float, C.c_int64, C.c_int64, C.c_int64,
                                           C.c_void_p, C.c_void_p]
    return _h


def available() -> bool:
    return _lib() is not None


def fill_tasks(base: int, n: int, lut64: np.ndarray, out: np.ndarray, chunk: int = 1 << 22):
    """Callables that together fill out[0:n] (for a caller-owned thread pool)."""
    lib = _lib()
    if lib is None:
        raise RuntimeError(f"{_LIB} not built (make -C oracle)")

    def one(s0):
        return lambda: lib.synth_f64_range(C.c_uint64(base), n, s0, min(chunk, n - s0), lut64.ctypes.data,
                                           out[s0:].ctypes.data)
    return [one(s0) for s0 in range(0, n, chunk)]


def fill_mix_tasks(base_key: int, delta_key: int, spread: float, n: int, lut16: np.ndarray, out: np.ndarray,
                   chunk: int = 1 << 22):
    """Callables filling out[0:n] with a clustered matrix: bf16_rn(b + spread*e) as f64."""
    lib = _lib()
    if lib is None:
        raise RuntimeError(f"{_LIB} not built (make -C oracle)")

    def one(s0):
        return lambda: lib.synth_mix_f64_range(C.c_uint64(base_key), C.c_uint64(delta_key), C.c_float(spread), n, s0,
                                               min(chunk, n - s0), lut16.ctypes.data, out[s0:].ctypes.data)
    return [one(s0) for s0 in range(0, n, chunk)]


def synth_f64(base: int, n: int, lut64: np.ndarray, out: np.ndarray | None = None, threads: int | None = None,
              chunk: int = 1 << 22) -> np.ndarray:
    """Values [0, n) of one matrix as float64: lut64[16-bit field of mix64(base + i/4)]."""
    lib = _lib()
    if lib is None:
        raise RuntimeError(f"{_LIB} not built (make -C oracle)")
    lut64 = np.ascontiguousarray(lut64, np.float64)
    out = np.empty(n, np.float64) if out is None else out
    threads = threads or len(os.sched_getaffinity(0))

    def work(s0):
        cnt = min(chunk, n - s0)
        lib.synth_f64_range(C.c_uint64(base), n, s0, cnt, lut64.ctypes.data, out[s0:].ctypes.data)

    with ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(work, range(0, n, chunk)))
    return out
