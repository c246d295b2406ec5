"""Adjusted Rand Index (Hubert & Arabie 1985).

PAPER.md §4.3 Eq. (11) (lines 354-360) and §5 (lines 372-374): the stability
measure and the recovery performance p(l_m) = ari(l, l_m) in [-1, 1].

    ARI = (sum_ij C(n_ij,2) - E) / (1/2 [sum_i C(a_i,2) + sum_j C(b_j,2)] - E),
    E   = sum_i C(a_i,2) sum_j C(b_j,2) / C(n,2)
with n_ij the contingency table and a, b its margins.  When the denominator is
zero the two partitions are both trivial; ARI := 1 if they are identical as
partitions, else 0 (reading R9).

ORACLE -- test infrastructure only (see oracle/__init__.py).
"""

from __future__ import annotations

import numpy as np


def _c2(x):
    x = np.asarray(x, dtype=np.float64)
    return x * (x - 1.0) / 2.0


def contingency(a, b) -> np.ndarray:
    a = np.asarray(a)
    b = np.asarray(b)
    _, ai = np.unique(a, return_inverse=True)
    _, bi = np.unique(b, return_inverse=True)
    t = np.zeros((ai.max() + 1, bi.max() + 1), dtype=np.int64)
    np.add.at(t, (ai, bi), 1)
    return t


def ari(a, b) -> float:
    n = len(a)
    t = contingency(a, b)
    sum_ij = _c2(t).sum()
    sa = _c2(t.sum(axis=1)).sum()
    sb = _c2(t.sum(axis=0)).sum()
    expected = sa * sb / _c2(n) if n > 1 else 0.0
    denom = 0.5 * (sa + sb) - expected
    if denom == 0.0:
        return 1.0 if (t.shape[0] == t.shape[1] and np.count_nonzero(t) == t.shape[0]) else 0.0
    return float((sum_ij - expected) / denom)
