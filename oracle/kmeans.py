"""k-means on the feature vectors, fp64.

PAPER.md §2.2 step 4 (lines 109-113) and §4.1 step 6 (lines 323-328): "Run
k-means ... with the Euclidean distance D~_ij = ||f~_i - f~_j||".  §5:
Matlab's k-means with replicates, whose default seeding is k-means++
(reading R8).  Decisions (argmin, D^2 sampling, best replicate) are
taken in fp64 on both sides (task rule: the paper's precision, Matlab double).

    seeding   : k-means++ (Arthur & Vassilvitskii 2007) with the uniforms u_0..u_{k-1}
                passed in: first centre floor(u_0 N); centre t is the smallest i
                with cumsum(D^2)_i > u_t * sum(D^2).
    Lloyd     : assign = argmin_c sum_q (x_iq - C_cq)^2 (lowest c on ties; the sum
                in ascending q);
                update = member mean, member sum correctly rounded (math.fsum),
                an empty cluster keeps its centre;
                stop when an assignment repeats or after max_iter updates.
    replicates: lowest inertia wins, ties -> lowest replicate index.

ORACLE -- test infrastructure only (see oracle/__init__.py).
"""

from __future__ import annotations

import math

import numpy as np


def sq_dists(X: np.ndarray, C: np.ndarray) -> np.ndarray:
    """D[i, c] = sum_q (X[i,q] - C[c,q])^2 in fp64, explicit differences, the sum
    taken term by term in ascending q (reading R8: the decision
    arithmetic is fixed so that both sides round identically)."""
    X = np.asarray(X, dtype=np.float64)
    C = np.asarray(C, dtype=np.float64)
    D = np.zeros((X.shape[0], C.shape[0]), dtype=np.float64)
    for c in range(C.shape[0]):
        acc = np.zeros(X.shape[0], dtype=np.float64)
        for q in range(X.shape[1]):
            diff = X[:, q] - C[c, q]
            acc += diff * diff
        D[:, c] = acc
    return D


def assign(X, C):
    D = sq_dists(X, C)
    lab = np.argmin(D, axis=1)            # first minimum on ties
    return lab.astype(np.int32), D[np.arange(D.shape[0]), lab]


def update(X, labels, C_prev):
    X = np.asarray(X, dtype=np.float64)
    k = C_prev.shape[0]
    C = np.array(C_prev, dtype=np.float64, copy=True)
    for c in range(k):
        m = labels == c
        cnt = int(m.sum())
        if cnt:
            M = X[m]
            # member mean with the member sum correctly rounded (math.fsum)
            C[c] = [math.fsum(M[:, q]) / cnt for q in range(X.shape[1])]
    return C


def kmeanspp(X, k: int, u: np.ndarray) -> np.ndarray:
    """Indices of the k-means++ seeds for uniforms u[0..k-1]."""
    X = np.asarray(X, dtype=np.float64)
    n = X.shape[0]
    idx = [min(int(np.floor(u[0] * n)), n - 1)]
    d2 = sq_dists(X, X[idx[0]][None, :])[:, 0]
    for t in range(1, k):
        cs = np.cumsum(d2)
        total = cs[-1]
        if total <= 0.0:
            nxt = min(int(np.floor(u[t] * n)), n - 1)
        else:
            nxt = int(np.searchsorted(cs, u[t] * total, side="right"))
            nxt = min(nxt, n - 1)
        idx.append(nxt)
        d2 = np.minimum(d2, sq_dists(X, X[nxt][None, :])[:, 0])
    return np.array(idx, dtype=np.int64)


def lloyd(X, C0, max_iter: int = 100):
    C = np.array(C0, dtype=np.float64, copy=True)
    labels, _ = assign(X, C)
    it = 0
    for it in range(1, max_iter + 1):
        C = update(X, labels, C)
        new, _ = assign(X, C)
        if np.array_equal(new, labels):
            break
        labels = new
    dmin = sq_dists(X, C)[np.arange(len(labels)), labels]
    return labels, C, float(np.sum(dmin)), it


def kmeans(X, k: int, uniforms_per_restart: np.ndarray, max_iter: int = 100):
    """Best of len(uniforms_per_restart) replicates; uniforms_per_restart[r] has k entries."""
    X = np.asarray(X, dtype=np.float64)
    best = None
    for r, u in enumerate(uniforms_per_restart):
        seeds = kmeanspp(X, k, u)
        labels, C, inertia, it = lloyd(X, X[seeds], max_iter)
        if best is None or inertia < best[2]:
            best = (labels, C, inertia, it, r, seeds)
    return best
