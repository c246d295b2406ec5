"""Seeded synthetic similarity graphs W as symmetric CSR.

PAPER.md §2 (lines 59-63): an undirected weighted graph with weighted adjacency
W, W_ij = W_ji >= 0.  §5 (lines 368-380) builds W as a kNN graph of a Gaussian
mixture; BASELINE.json adds stochastic-block-model (SBM) graphs.  Nodes of an
SBM are numbered community by community (contiguous blocks), so ``labels`` is
non-decreasing.

CSR convention used everywhere in this repo:
    row_ptr  int64[N+1], col_idx int32[nnz] (sorted within each row, no
    diagonal), values float32[nnz] or None (None == every stored weight is 1,
    "pattern" CSR used for the unit-weight SBM graphs).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class CSRGraph:
    n: int
    row_ptr: np.ndarray            # int64 [n+1]
    col_idx: np.ndarray            # int32 [nnz]
    values: np.ndarray | None      # float32 [nnz] or None (unit weights)
    labels: np.ndarray | None = None   # planted community / mixture label per node
    meta: dict = field(default_factory=dict)

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def weights(self, dtype=np.float64) -> np.ndarray:
        if self.values is None:
            return np.ones(self.nnz, dtype=dtype)
        return self.values.astype(dtype)

    def degrees(self) -> np.ndarray:
        return np.diff(self.row_ptr)


# ----------------------------------------------------------------------------
# CSR assembly
# ----------------------------------------------------------------------------

def from_edges(n: int, a: np.ndarray, b: np.ndarray, w: np.ndarray | None = None,
               labels=None, meta=None) -> CSRGraph:
    """Symmetric CSR from an undirected edge list (a_e, b_e, w_e), a_e != b_e.

    Duplicate undirected edges are merged (first weight kept)."""
    a = np.asarray(a, dtype=np.int64)
    b = np.asarray(b, dtype=np.int64)
    if np.any(a == b):
        raise ValueError("self loops are not allowed (W has zero diagonal)")
    lo = np.minimum(a, b)
    hi = np.maximum(a, b)
    key = lo * n + hi
    key, first = np.unique(key, return_index=True)
    lo = key // n
    hi = key % n
    if w is not None:
        w = np.asarray(w, dtype=np.float32)[first]
    rows = np.concatenate([lo, hi])
    cols = np.concatenate([hi, lo])
    order = np.argsort(rows * n + cols, kind="stable")
    rows = rows[order]
    cols = cols[order]
    vals = None
    if w is not None:
        vals = np.concatenate([w, w])[order]
    counts = np.bincount(rows, minlength=n)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    return CSRGraph(n=n, row_ptr=row_ptr, col_idx=cols.astype(np.int32), values=vals,
                    labels=None if labels is None else np.asarray(labels, dtype=np.int32),
                    meta=dict(meta or {}))


def _connect_isolated(n, lo, hi, labels, rng):
    """Attach degree-0 nodes to a random node of their own community (PAPER.md
    line 79 only considers connected graphs)."""
    deg = np.bincount(lo, minlength=n) + np.bincount(hi, minlength=n)
    iso = np.nonzero(deg == 0)[0]
    if iso.size == 0:
        return lo, hi
    extra_a, extra_b = [], []
    for v in iso:
        same = np.nonzero(labels == labels[v])[0] if labels is not None else np.arange(n)
        cand = same[same != v]
        if cand.size == 0:
            cand = np.setdiff1d(np.arange(n), [v])
        u = int(cand[rng.integers(cand.size)])
        extra_a.append(min(u, v))
        extra_b.append(max(u, v))
    return (np.concatenate([lo, np.array(extra_a, dtype=np.int64)]),
            np.concatenate([hi, np.array(extra_b, dtype=np.int64)]))


def _connect_components(g: CSRGraph, rng) -> CSRGraph:
    """Join every non-giant connected component to the giant one by one edge."""
    import scipy.sparse as sp
    from scipy.sparse.csgraph import connected_components
    m = sp.csr_matrix((np.ones(g.nnz), g.col_idx, g.row_ptr), shape=(g.n, g.n))
    ncomp, comp = connected_components(m, directed=False)
    if ncomp == 1:
        return g
    giant = np.argmax(np.bincount(comp))
    giant_nodes = np.nonzero(comp == giant)[0]
    rows = np.repeat(np.arange(g.n, dtype=np.int64), np.diff(g.row_ptr))
    keep = rows < g.col_idx
    a = [rows[keep]]
    b = [g.col_idx[keep].astype(np.int64)]
    w = [g.values[keep]] if g.values is not None else None
    # the lowest node of every other component, joined to a uniformly drawn giant node
    _, first = np.unique(comp, return_index=True)
    first = first[np.arange(ncomp) != giant].astype(np.int64)
    u = giant_nodes[rng.integers(giant_nodes.size, size=first.size)].astype(np.int64)
    a.append(np.minimum(u, first))
    b.append(np.maximum(u, first))
    if w is not None:
        w.append(np.ones(first.size, dtype=np.float32))
    return from_edges(g.n, np.concatenate(a), np.concatenate(b),
                      None if w is None else np.concatenate(w), labels=g.labels, meta=g.meta)


# ----------------------------------------------------------------------------
# Stochastic block model (BASELINE.json configs 0, 2, 3, 4)
# ----------------------------------------------------------------------------

def community_sizes(n: int, k: int, kind: str = "equal", exponent: float = 2.0,
                    min_size: int = 1000, seed: int = 0) -> np.ndarray:
    if kind == "equal":
        sizes = np.full(k, n // k, dtype=np.int64)
        sizes[: n % k] += 1
        return sizes
    if kind == "powerlaw":
        # excess sizes ~ Pareto tail p(s) ~ s^-exponent, rescaled so that the
        # minimum is min_size and the total is n.
        if k * min_size > n:
            raise ValueError("k*min_size exceeds n")
        rng = np.random.default_rng(np.random.PCG64(seed ^ 0x51ED))
        w = min_size * (rng.pareto(exponent - 1.0, size=k) + 1.0) - min_size
        w = np.maximum(w, 0.0)
        if w.sum() == 0:
            w[:] = 1.0
        extra = np.floor((n - k * min_size) * w / w.sum()).astype(np.int64)
        sizes = min_size + extra
        sizes[np.argmax(sizes)] += n - sizes.sum()
        return np.sort(sizes)[::-1].copy()
    raise ValueError(kind)


def sbm(n: int, k: int, avg_degree: float, eps: float, sizes: str = "equal",
        exponent: float = 2.0, min_size: int = 1000, seed: int = 0,
        check_connected: bool | None = None) -> CSRGraph:
    """SBM with q_out = eps * q_in and expected mean degree ``avg_degree``.

    Edge counts per block are Binomial; endpoints are uniform within the block;
    duplicate pairs are merged (a ~avg_degree/N relative loss).  Unit weights.
    """
    rng = np.random.default_rng(np.random.PCG64(seed))
    sz = community_sizes(n, k, sizes, exponent, min_size, seed)
    off = np.zeros(k + 1, dtype=np.int64)
    np.cumsum(sz, out=off[1:])
    labels = np.repeat(np.arange(k, dtype=np.int32), sz)
    szf = sz.astype(np.float64)
    intra_pairs = szf * (szf - 1.0) / 2.0
    inter_pairs = (float(n) ** 2 - np.sum(szf ** 2)) / 2.0
    # E[sum of degrees] = 2 (q_in * intra + q_out * inter) = avg_degree * n
    q_in = avg_degree * n / (2.0 * (intra_pairs.sum() + eps * inter_pairs))
    q_out = eps * q_in
    if q_in > 1.0:
        raise ValueError("avg_degree too large for these community sizes")

    m_c = rng.binomial(intra_pairs.astype(np.int64), q_in)
    comm = np.repeat(np.arange(k), m_c)
    u = off[comm] + (rng.random(comm.size) * sz[comm]).astype(np.int64)
    v = off[comm] + (rng.random(comm.size) * sz[comm]).astype(np.int64)
    keep = u != v
    a_in, b_in = u[keep], v[keep]

    m_out = int(rng.binomial(int(inter_pairs), q_out)) if k > 1 else 0
    a_out = np.empty(0, dtype=np.int64)
    b_out = np.empty(0, dtype=np.int64)
    need = m_out
    while need > 0:
        u = rng.integers(0, n, size=need, dtype=np.int64)
        v = rng.integers(0, n, size=need, dtype=np.int64)
        keep = labels[u] != labels[v]
        a_out = np.concatenate([a_out, u[keep]])
        b_out = np.concatenate([b_out, v[keep]])
        need = m_out - a_out.size

    a = np.concatenate([a_in, a_out])
    b = np.concatenate([b_in, b_out])
    lo = np.minimum(a, b)
    hi = np.maximum(a, b)
    lo, hi = _connect_isolated(n, lo, hi, labels, rng)
    g = from_edges(n, lo, hi, None, labels=labels,
                   meta=dict(kind="sbm", k=k, avg_degree=avg_degree, eps=eps, sizes=sizes,
                             q_in=q_in, q_out=q_out, seed=seed))
    if check_connected is None:
        check_connected = True     # PAPER.md l.79 considers connected graphs (all sizes, round 2)
    if check_connected:
        g = _connect_components(g, rng)
    return g


def chung_lu(n: int, avg_degree: float, exponent: float, seed: int = 0, max_degree: int | None = None) -> CSRGraph:
    """Power-law-degree graph (Chung-Lu): node i has expected degree w_i proportional to
    (i + i0)^(-1/(exponent - 1)), scaled to mean ``avg_degree`` (w_0 capped at ``max_degree``,
    default sqrt(n) * avg_degree); the m = n * avg_degree / 2 edges join endpoints drawn
    independently with probability w / sum(w), self loops dropped and duplicates merged (so
    realised degrees of the largest hubs fall a little short of w).  Node ids are shuffled so
    hubs are spread over the tiles.  Unit weights.  (North_star: the traversal must cope
    with the degree distribution.)"""
    rng = np.random.default_rng(np.random.PCG64(seed))
    beta = 1.0 / (exponent - 1.0)
    i = np.arange(n, dtype=np.float64)
    w = (i + 1.0) ** (-beta)
    w *= avg_degree * n / w.sum()
    cap = float(max_degree if max_degree is not None else np.sqrt(n) * avg_degree)
    for _ in range(20):                      # cap the largest weights, keep the mean
        over = w > cap
        if not over.any():
            break
        w[over] = cap
        w *= avg_degree * n / w.sum()
    p = w / w.sum()
    m = int(round(n * avg_degree / 2.0))
    cdf = np.cumsum(p)
    a = np.searchsorted(cdf, rng.random(m) * cdf[-1], side="right")
    b = np.searchsorted(cdf, rng.random(m) * cdf[-1], side="right")
    a = np.minimum(a, n - 1)
    b = np.minimum(b, n - 1)
    keep = a != b
    perm = rng.permutation(n)
    g = from_edges(n, perm[a[keep]], perm[b[keep]], None,
                   meta=dict(kind="chung_lu", avg_degree=avg_degree, exponent=exponent, seed=seed))
    return g


# ----------------------------------------------------------------------------
# Gaussian-mixture kNN graph (§5; BASELINE.json config 1)
# ----------------------------------------------------------------------------

def gmm_points(n: int, dim: int, n_comp: int, sigma: float = 1.0, center_range: float = 10.0,
               seed: int = 0):
    rng = np.random.default_rng(np.random.PCG64(seed))
    centers = rng.uniform(0.0, center_range, size=(n_comp, dim))
    labels = rng.integers(0, n_comp, size=n).astype(np.int32)
    x = centers[labels] + sigma * rng.standard_normal((n, dim))
    return x, labels, centers


def gmm_knn(n: int = 20_000, dim: int = 10, n_comp: int = 10, knn: int = 10, sigma: float = 1.0,
            center_range: float = 10.0, seed: int = 0, weighting: str = "gaussian") -> CSRGraph:
    """Union-symmetrised kNN graph of a Gaussian mixture.

    Weights exp(-||x_i - x_j||^2 / s^2) with s = mean kNN distance (BASELINE.json
    config 1), or unit weights with ``weighting='binary'``.
    """
    from scipy.spatial import cKDTree
    x, labels, _ = gmm_points(n, dim, n_comp, sigma, center_range, seed)
    tree = cKDTree(x)
    dist, idx = tree.query(x, k=knn + 1)
    # drop self (first column may not be self for duplicate points; remove i==j)
    rows = np.repeat(np.arange(n, dtype=np.int64), knn + 1)
    cols = idx.reshape(-1).astype(np.int64)
    d = dist.reshape(-1)
    keep = rows != cols
    rows, cols, d = rows[keep], cols[keep], d[keep]
    # keep exactly knn neighbours per node
    rank = np.zeros_like(rows)
    _, start = np.unique(rows, return_index=True)
    rank = np.arange(rows.size) - np.repeat(start, np.diff(np.append(start, rows.size)))
    keep = rank < knn
    rows, cols, d = rows[keep], cols[keep], d[keep]
    s = float(d.mean())
    w = np.exp(-(d ** 2) / (s ** 2)).astype(np.float32) if weighting == "gaussian" else None
    g = from_edges(n, rows, cols, w, labels=labels,
                   meta=dict(kind="gmm_knn", dim=dim, n_comp=n_comp, knn=knn, kernel_sigma=s,
                             seed=seed))
    rng = np.random.default_rng(np.random.PCG64(seed + 1))
    return _connect_components(g, rng)


def permute(g: CSRGraph, perm: np.ndarray) -> CSRGraph:
    """Relabel node perm[i] as i (new CSR, columns sorted per row); labels follow."""
    n = g.n
    inv = np.empty(n, dtype=np.int64)
    inv[perm] = np.arange(n, dtype=np.int64)
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(g.row_ptr))
    a, b = inv[rows], inv[g.col_idx.astype(np.int64)]
    order = np.lexsort((b, a))
    a, b = a[order], b[order]
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(row_ptr, a + 1, 1)
    row_ptr = np.cumsum(row_ptr)
    vals = None if g.values is None else g.values[order]
    labels = None if g.labels is None else g.labels[perm]
    return CSRGraph(n=n, row_ptr=row_ptr, col_idx=b.astype(np.int32), values=vals, labels=labels,
                    meta=dict(g.meta, permuted=True))


def rcm_order(g: CSRGraph) -> CSRGraph:
    """Reverse Cuthill-McKee relabelling (scipy.sparse.csgraph): neighbours get nearby
    indices, so the rows a tile gathers are close together in memory."""
    import scipy.sparse as sp
    from scipy.sparse.csgraph import reverse_cuthill_mckee
    A = sp.csr_matrix((np.ones(g.nnz, dtype=np.int8), g.col_idx, g.row_ptr), shape=(g.n, g.n))
    perm = np.asarray(reverse_cuthill_mckee(A, symmetric_mode=True), dtype=np.int64)
    out = permute(g, perm)
    out.meta["order"] = "rcm"
    return out


# ----------------------------------------------------------------------------
# Small fixtures with closed-form spectra (tests)
# ----------------------------------------------------------------------------

def ring(n: int, w: float | None = None) -> CSRGraph:
    a = np.arange(n, dtype=np.int64)
    b = (a + 1) % n
    return from_edges(n, a, b, None if w is None else np.full(n, w, np.float32),
                      meta=dict(kind="ring"))


def path(n: int, w: float | None = None) -> CSRGraph:
    a = np.arange(n - 1, dtype=np.int64)
    return from_edges(n, a, a + 1, None if w is None else np.full(n - 1, w, np.float32),
                      meta=dict(kind="path"))


def complete(n: int) -> CSRGraph:
    a, b = np.triu_indices(n, 1)
    return from_edges(n, a, b, None, meta=dict(kind="complete"))


def star(leaves: int) -> CSRGraph:
    return from_edges(leaves + 1, np.zeros(leaves, np.int64), np.arange(1, leaves + 1),
                      None, meta=dict(kind="star"))


def two_cliques(m: int, bridge_w: float = 0.1) -> CSRGraph:
    """Two m-cliques (unit weights) joined by one edge of weight bridge_w."""
    a1, b1 = np.triu_indices(m, 1)
    a = np.concatenate([a1, a1 + m, [m - 1]])
    b = np.concatenate([b1, b1 + m, [m]])
    w = np.concatenate([np.ones(a1.size * 2), [bridge_w]]).astype(np.float32)
    labels = np.repeat([0, 1], m)
    return from_edges(2 * m, a, b, w, labels=labels, meta=dict(kind="two_cliques"))


def random_connected(n: int, p: float, seed: int, weighted: bool = True) -> CSRGraph:
    """Erdos-Renyi graph plus a random spanning path (so it is connected),
    with U[0.5, 1.5] weights if ``weighted``."""
    rng = np.random.default_rng(np.random.PCG64(seed))
    a, b = np.triu_indices(n, 1)
    keep = rng.random(a.size) < p
    perm = rng.permutation(n)
    a = np.concatenate([a[keep], perm[:-1]])
    b = np.concatenate([b[keep], perm[1:]])
    w = rng.uniform(0.5, 1.5, size=a.size).astype(np.float32) if weighted else None
    return from_edges(n, a, b, w, meta=dict(kind="er", p=p, seed=seed))
