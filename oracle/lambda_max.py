"""Estimate of the largest Laplacian eigenvalue lambda_N.

PAPER.md §4.1 step 1 (line 309): "Estimate [trefethen1997numerical] L's largest
eigenvalue lambda_N (necessary for steps 2 and 3)."  The cited textbook method
is the power iteration with Rayleigh quotient (Trefethen & Bau, Lecture 27).
Because the Chebyshev domain [0, lambda_max] must contain the whole spectrum
(reading R3), the returned bound is the Rayleigh quotient inflated by
(1 + margin).

ORACLE -- test infrastructure only (see oracle/__init__.py).
"""

from __future__ import annotations

import numpy as np


def power_iteration(L, x0: np.ndarray, iters: int = 500):
    """Plain power iteration: v <- L v / ||L v||; returns the Rayleigh quotient
    v^T L v of the last iterate and the iterate."""
    v = np.asarray(x0, dtype=np.float64)
    v = v / np.linalg.norm(v)
    rq = 0.0
    for _ in range(iters):
        w = L @ v
        rq = float(v @ w)
        nrm = np.linalg.norm(w)
        if nrm == 0.0:
            return 0.0, v
        v = w / nrm
    return rq, v


def lambda_max_bound(L, x0: np.ndarray, iters: int = 500, margin: float = 0.01) -> float:
    """Upper bound used as the Chebyshev domain end: (1 + margin) * Rayleigh quotient."""
    rq, _ = power_iteration(L, x0, iters)
    return (1.0 + margin) * rq


def lambda_max_exact(L) -> float:
    """Exact lambda_N by a dense symmetric eigensolver (pins / small graphs)."""
    import scipy.sparse as sp
    A = L.toarray() if sp.issparse(L) else np.asarray(L)
    return float(np.linalg.eigvalsh(A)[-1])
