"""Ideal low-pass graph filter and its fast (polynomial) approximation.

PAPER.md §2.3 Eq. (2) (lines 126-130): h_{lambda_c}(lambda) = 1 if lambda <= lambda_c else 0,
H = chi diag(h(lambda_l)) chi^T (line 122).

PAPER.md §2.4 Eq. (3) (lines 135-147): Hx ~= sum_{l=0}^m alpha_l L^l x = F^m_h x, a
polynomial of order m in L that "only requires matrix-vector multiplication",
following [shuman_DCOSS2011], whose polynomial is the truncated Chebyshev
expansion of h on [0, lambda_max] evaluated by the three-term recurrence
(reading R1: the polynomial basis is Chebyshev, as BASELINE.json's
north_star states).  Optional Jackson damping (reading R2).

Notation:
    x = 2 lambda / lambda_max - 1  maps [0, lambda_max] to [-1, 1]
    L~ = (2 / lambda_max) L - I
    h(x) ~= sum_{j=0}^{p} g_j c_j T_j(x)        (g_j = 1 without damping)
    T_0 = R,  T_1 = L~ R,  T_{j+1} = 2 L~ T_j - T_{j-1}
    Y = F R = sum_j g_j c_j T_j

ORACLE -- test infrastructure only (see oracle/__init__.py).
"""

from __future__ import annotations

import numpy as np


def ideal_lowpass(lam, lambda_c: float):
    """Eq. (2): 1 where lambda <= lambda_c, else 0."""
    return (np.asarray(lam, dtype=np.float64) <= lambda_c).astype(np.float64)


def lowpass_coeffs(lambda_c: float, lambda_max: float, order: int) -> np.ndarray:
    """Chebyshev coefficients c_0..c_p of h_{lambda_c} on [0, lambda_max].

    With x = cos(theta), h(cos theta) = 1 iff theta >= theta_c = arccos(a),
    a = 2 lambda_c / lambda_max - 1.  The Chebyshev series coefficients
    (2/pi) int_0^pi h(cos t) cos(j t) dt, with the j=0 term halved, are
        c_0 = 1 - theta_c / pi,      c_j = -2 sin(j theta_c) / (pi j)   (j >= 1).
    """
    if order < 0:
        raise ValueError("order must be >= 0")
    a = np.clip(2.0 * lambda_c / lambda_max - 1.0, -1.0, 1.0)
    theta_c = np.arccos(a)
    c = np.empty(order + 1, dtype=np.float64)
    c[0] = 1.0 - theta_c / np.pi
    j = np.arange(1, order + 1, dtype=np.float64)
    c[1:] = -2.0 * np.sin(j * theta_c) / (np.pi * j)
    return c


def jackson(order: int) -> np.ndarray:
    """Jackson damping factors g_0..g_p for a (p+1)-term Chebyshev series
    (kernel polynomial method, Weisse et al. 2006, with M = p+1 moments):
        g_j = [(M - j + 1) cos(pi j/(M+1)) + sin(pi j/(M+1)) cot(pi/(M+1))] / (M+1).
    """
    M = order + 1
    j = np.arange(order + 1, dtype=np.float64)
    q = np.pi / (M + 1)
    return ((M - j + 1) * np.cos(q * j) + np.sin(q * j) / np.tan(q)) / (M + 1)


def filter_coeffs(lambda_c: float, lambda_max: float, order: int, damping: bool) -> np.ndarray:
    """The coefficients g_j c_j actually applied by F^p."""
    c = lowpass_coeffs(lambda_c, lambda_max, order)
    return c * jackson(order) if damping else c


def poly_eval(lam, coeffs: np.ndarray, lambda_max: float):
    """Scalar polynomial p(lambda) = sum_j coeffs_j T_j(x), T_j(x) = cos(j arccos x)
    (trigonometric form; the recurrence is NOT used here)."""
    x = np.clip(2.0 * np.asarray(lam, dtype=np.float64) / lambda_max - 1.0, -1.0, 1.0)
    t = np.arccos(x)
    j = np.arange(len(coeffs), dtype=np.float64)
    return np.cos(np.multiply.outer(t, j)) @ coeffs


def order_grid(ratio: float, theta: float = 0.1, n_grid: int = 10000) -> np.ndarray:
    """Points of [0, 1] where the §2.4 criterion (Eq. (4), l.151-156) is checked for
    h_{ratio} = h_{lambda_c/lambda_N} on [0, 1] (l.157-159: the normalised filter depends on
    the ratio only): the uniform n_grid-point grids i/(n_grid-1) of [0, 1] and of
    [0, min(1, 2 ratio)] (the second resolves the neighbourhood of the cut whatever the
    ratio), minus the transition band [ratio(1-theta), ratio(1+theta)] (reading R18:
    the sup over all of [0, lambda_N] is >= 1/2 for any polynomial at the jump)."""
    i = np.arange(n_grid, dtype=np.float64) / (n_grid - 1)
    lam = np.union1d(i, i * min(1.0, 2.0 * ratio))
    keep = (lam < ratio * (1.0 - theta)) | (lam > ratio * (1.0 + theta))
    return lam[keep]


def approx_error(ratio: float, order: int, damping: bool, theta: float = 0.1,
                 n_grid: int = 10000) -> float:
    """sup over order_grid of |h_{ratio}(lambda) - p_m(lambda)|, p_m the order-m polynomial
    the filter applies (filter_coeffs on [0, 1]), evaluated in trigonometric form."""
    lam = order_grid(ratio, theta, n_grid)
    p = poly_eval(lam, filter_coeffs(ratio, 1.0, order, damping), 1.0)
    return float(np.max(np.abs(ideal_lowpass(lam, ratio) - p)))


def minimal_order(ratio: float, delta: float, damping: bool, m_max: int, theta: float = 0.1,
                  n_grid: int = 10000):
    """m*(lambda_c/lambda_N; delta) (§2.4 l.151-162, §4.1 step 3 l.312): the smallest
    m in 1..m_max with approx_error <= delta, tried in increasing m; None if there is none."""
    for m in range(1, m_max + 1):
        if approx_error(ratio, m, damping, theta, n_grid) <= delta:
            return m
    return None


def cheb_filter(L, R: np.ndarray, coeffs: np.ndarray, lambda_max: float) -> np.ndarray:
    """Y = sum_j coeffs_j T_j(L~) R by the three-term recurrence, fp64.

    One sparse product L @ T per order (cost O(m(|E|+N)))."""
    T0 = np.asarray(R, dtype=np.float64)
    p = len(coeffs) - 1
    a = 2.0 / lambda_max

    def Lt(X):                       # L~ X = (2/lambda_max) L X - X
        return a * (L @ X) - X

    Y = coeffs[0] * T0
    if p == 0:
        return Y
    T1 = Lt(T0)
    Y = Y + coeffs[1] * T1
    for j in range(1, p):
        T2 = 2.0 * Lt(T1) - T0
        Y = Y + coeffs[j + 1] * T2
        T0, T1 = T1, T2
    return Y


def lowpass_filter(L, R, lambda_c: float, lambda_max: float, order: int, damping: bool = False):
    """F^p_{lambda_c} R (§4.1 steps 3 and 5, Eq. (10))."""
    return cheb_filter(L, R, filter_coeffs(lambda_c, lambda_max, order, damping), lambda_max)


def ideal_filter_dense(L_dense: np.ndarray, R: np.ndarray, lambda_c: float) -> np.ndarray:
    """Exact H_{lambda_c} R = chi diag(h(lambda)) chi^T R by dense eigendecomposition
    (small graphs only)."""
    lam, chi = np.linalg.eigh(L_dense)
    return chi @ (ideal_lowpass(lam, lambda_c)[:, None] * (chi.T @ R))
