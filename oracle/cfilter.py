"""ctypes loader of oracle/cfilter.c (plain C + OpenMP fp64 Chebyshev filter).

ORACLE -- test infrastructure only (see oracle/__init__.py).  Same definition as
chebyshev.cheb_filter (§2.4 Eq. (3) l.135-147, §4.1 step 5 Eq. (10) l.321),
rows of each recurrence step split across host threads.  The shared object is built with
gcc on first use (``build()``; __graft_entry__.build() calls it too).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "cfilter.c")
_LIB = os.path.join(_HERE, "libcfilter.so")
_lib = None


def build() -> str:
    if not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.run(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-o", _LIB, _SRC], check=True)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        _lib.oracle_cheb_filter.argtypes = [ctypes.c_int64, P, P, P, ctypes.c_int, P, P, ctypes.c_int,
                                            ctypes.c_double, P, ctypes.c_int]
        _lib.oracle_cheb_filter.restype = ctypes.c_int
        _lib.oracle_num_threads.restype = ctypes.c_int
    return _lib


def num_threads() -> int:
    return int(_load().oracle_num_threads())


def cheb_filter(g, R: np.ndarray, coeffs: np.ndarray, lambda_max: float, nthreads: int = 0) -> np.ndarray:
    """Y = sum_j coeffs_j T_j(L~) R for the graph g (scinputs CSR of W), fp64."""
    lib = _load()
    R = np.ascontiguousarray(R, dtype=np.float64)
    if R.ndim == 1:
        R = R[:, None]
    n, k = R.shape
    rp = np.ascontiguousarray(g.row_ptr, dtype=np.int64)
    col = np.ascontiguousarray(g.col_idx, dtype=np.int32)
    val = None if g.values is None else np.ascontiguousarray(g.values, dtype=np.float64)
    d = np.ascontiguousarray(coeffs, dtype=np.float64)
    Y = np.empty_like(R)
    rc = lib.oracle_cheb_filter(n, rp.ctypes.data, col.ctypes.data, 0 if val is None else val.ctypes.data, k,
                                R.ctypes.data, d.ctypes.data, len(d) - 1, float(lambda_max), Y.ctypes.data,
                                int(nthreads))
    if rc != 0:
        raise MemoryError("oracle_cheb_filter: allocation failed")
    return Y
