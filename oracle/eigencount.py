"""Eigenvalue count below a cut and dichotomous estimate of lambda_k.

PAPER.md §3.2: "we estimate the spectrum's cumulative density
function as in Section VB of [shuman_TSP2015] ... Given a graph Laplacian L and
a 'cutting frequency' lambda_c, the algorithm estimates the number of
eigenvalues inferior to lambda_c.  Using a dichotomous procedure on
[0, lambda_N], we obtain an estimate of lambda_k, noted lambda~_k."

The cited estimator filters random signals with the ideal low-pass h_{lambda_c}
and measures the energy that passes: for R with i.i.d. N(0, 1/n_probe) entries
and n_probe columns, E ||H_{lambda_c} R||_F^2 = trace(H^2) = #{l : lambda_l <= lambda_c}.
H is replaced by its fast filter F^p (reading R5).  The dichotomy keeps
count(lo) < k <= count(hi) (reading R6).

ORACLE -- test infrastructure only (see oracle/__init__.py).
"""

from __future__ import annotations

import numpy as np

from . import chebyshev


def count_below(L, lambda_c: float, lambda_max: float, order: int, R: np.ndarray,
                damping: bool = True) -> float:
    """||F^p_{lambda_c} R||_F^2 (R entries ~ N(0, 1/n_probe))."""
    Y = chebyshev.lowpass_filter(L, R, lambda_c, lambda_max, order, damping)
    return float(np.sum(Y * Y))


def estimate_lambda_k(L, k: int, lambda_max: float, order: int, R: np.ndarray,
                      damping: bool = True, max_iter: int = 30, rtol: float = 1e-3):
    """Dichotomy on [0, lambda_max]; returns (lambda~_k = hi, count(hi), trace).

    A cut is 'at or above lambda_k' when its count rounds to >= k, i.e.
    count >= k - 1/2."""
    lo, hi = 0.0, float(lambda_max)
    c_hi = float("nan")
    trace = []
    for _ in range(max_iter):
        mid = 0.5 * (lo + hi)
        c = count_below(L, mid, lambda_max, order, R, damping)
        trace.append((mid, c))
        if c >= k - 0.5:
            hi, c_hi = mid, c
        else:
            lo = mid
        if hi - lo <= rtol * lambda_max:
            break
    return hi, c_hi, trace
