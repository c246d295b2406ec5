"""Stability measure gamma(k), §4.3 Eq. (11) (lines 351-362).

For each k, J clusterings C^1..C^J from J realisations of the random signals;
gamma(k) is "the mean of the Adjusted Rand Index similarity between all pairs
of clusterings".  Eq. (11) writes 2/(J(J-1)) sum_{i != j}; the normalisation
2/(J(J-1)) is one over the number of UNORDERED pairs, so the sum runs over
i < j (reading R7).  k* = argmax gamma, smallest k on ties.

ORACLE -- test infrastructure only (see oracle/__init__.py).
"""

from __future__ import annotations

import itertools

from . import ari as _ari


def gamma(labelings) -> float:
    J = len(labelings)
    if J < 2:
        raise ValueError("J >= 2 required")
    tot = 0.0
    for i, j in itertools.combinations(range(J), 2):
        tot += _ari.ari(labelings[i], labelings[j])
    return 2.0 * tot / (J * (J - 1))


def k_star(gammas: dict) -> int:
    best = max(gammas.values())
    return min(k for k, g in gammas.items() if g == best)
