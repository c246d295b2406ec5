"""The accelerated spectral clustering algorithm, §4.1 (lines 303-329).

    1. lambda_N estimate                        (lambda_max.lambda_max_bound)
    2. lambda~_k by eigencount dichotomy        (eigencount.estimate_lambda_k)
    3. m = m*(lambda~_k/lambda_N; delta)         (chebyshev.minimal_order, when order < 0)
       polynomial approximation of h_{lambda~_k} (chebyshev.filter_coeffs)
    4. R: N x eta Gaussian, variance 1/eta      (scinputs.signals, passed in)
    5. f~_i^T = delta_i^T F R                   (chebyshev.cheb_filter, Eq. (10))
    6. k-means on the f~_i                      (kmeans.kmeans)

Optional per-row normalisation f~_i / ||f~_i|| before step 6 (BASELINE.json
north_star item (5); not in PAPER.md §4.1 -- DESIGN.md reading R10).

ORACLE -- test infrastructure only (see oracle/__init__.py).
"""

from __future__ import annotations

import numpy as np

from . import chebyshev, eigencount, kmeans, laplacian, lambda_max


def normalize_rows(F: np.ndarray) -> np.ndarray:
    """f_i / ||f_i||_2 (rows with zero norm are left at zero)."""
    F = np.asarray(F, dtype=np.float64)
    nrm = np.sqrt(np.sum(F * F, axis=1))
    out = np.zeros_like(F)
    nz = nrm > 0
    out[nz] = F[nz] / nrm[nz, None]
    return out


def accelerated_sc(g, k: int, R: np.ndarray, R_probe: np.ndarray, order: int, damping: bool,
                   kmeans_uniforms: np.ndarray, lambda_max_value: float | None = None,
                   x0: np.ndarray | None = None, normalize: bool = False, max_iter: int = 100,
                   bisect_iter: int = 30, bisect_rtol: float = 1e-3):
    L = laplacian.laplacian(g)
    if lambda_max_value is None:
        lambda_max_value = lambda_max.lambda_max_bound(L, x0)
    est_order = abs(order)
    lam_k, count_k, _ = eigencount.estimate_lambda_k(L, k, lambda_max_value, est_order, R_probe,
                                                     True, bisect_iter, bisect_rtol)
    # step 3 (l.312): order < 0 -> m = m*(lambda~_k/lambda_N; delta = 0.1) (l.162, reading R18)
    filt_order = order
    if order < 0:
        filt_order = chebyshev.minimal_order(min(1.0, lam_k / lambda_max_value), 0.1, damping, 2000) or 2000
    Y = chebyshev.lowpass_filter(L, R, lam_k, lambda_max_value, filt_order, damping)
    feats = normalize_rows(Y) if normalize else Y
    labels, C, inertia, it, rep, seeds = kmeans.kmeans(feats, k, kmeans_uniforms, max_iter)
    return dict(lambda_max=lambda_max_value, lambda_k=lam_k, count_k=count_k, features=Y,
                labels=labels, inertia=inertia, iters=it, replicate=rep, order=filt_order)
