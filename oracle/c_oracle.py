"""ctypes wrapper of oracle/build/libpsim_oracle.so (TEST / BASELINE ONLY)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "build" / "libpsim_oracle.so"
_lib = None


def build() -> Path:
    if not LIB.exists() or LIB.stat().st_mtime < (HERE / "psim_oracle.c").stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        h = C.CDLL(str(LIB))
        i64, vp = C.c_int64, C.c_void_p
        for sfx in ("f64", "f32"):
            f = getattr(h, f"oracle_mgemm_{sfx}")
            f.argtypes = [vp, i64, vp, i64, i64, i64, i64, vp, i64, C.c_int]
            f.restype = None
            f = getattr(h, f"oracle_czek2_{sfx}")
            f.argtypes = [vp, i64, i64, i64, vp, vp, C.c_int]
            f.restype = i64
        h.oracle_mix64.argtypes = [C.c_uint64]
        h.oracle_mix64.restype = C.c_uint64
        _lib = h
    return _lib


def threads() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()


def _sfx(a: np.ndarray) -> str:
    return "f64" if a.dtype == np.float64 else "f32"


def mgemm(W: np.ndarray, V: np.ndarray, nthreads: int | None = None) -> np.ndarray:
    """Blocked min-plus (mingemm.py:94-117) on Fortran (n_f, m) x (n_f, n) inputs."""
    W = np.asfortranarray(W)
    V = np.asfortranarray(V, dtype=W.dtype)
    n_f, m = W.shape
    n = V.shape[1]
    M = np.zeros((m, n), dtype=W.dtype, order="F")
    getattr(lib(), f"oracle_mgemm_{_sfx(W)}")(
        W.ctypes.data, n_f, V.ctypes.data, n_f, n_f, m, n, M.ctypes.data, m,
        nthreads or threads())
    return M


def czek2(V: np.ndarray, nthreads: int | None = None):
    """Full single-rank 2-way run: (canonical values, checksum hex, degenerate count)."""
    V = np.asfortranarray(V)
    n_f, n_v = V.shape
    vals = np.empty(n_v * (n_v - 1) // 2, dtype=V.dtype)
    cks = np.zeros(2, dtype=np.uint64)
    deg = getattr(lib(), f"oracle_czek2_{_sfx(V)}")(
        V.ctypes.data, n_f, n_f, n_v, vals.ctypes.data, cks.ctypes.data, nthreads or threads())
    value = (int(cks[1]) << 64) | int(cks[0])
    return vals, format(value, "032x"), int(deg)
