"""Combinatorial Laplacian, §2.1 lines 66-72.

    L = S - W,   S = diag(s),   s_i = sum_{j != i} W_ij   (strength of node i)

ORACLE -- test infrastructure only (see oracle/__init__.py).
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp


def adjacency(g) -> sp.csr_matrix:
    """W as an fp64 scipy CSR matrix from a ``scinputs.CSRGraph``."""
    return sp.csr_matrix((g.weights(np.float64), g.col_idx.astype(np.int64), g.row_ptr),
                         shape=(g.n, g.n))


def strengths(W: sp.csr_matrix) -> np.ndarray:
    """s_i = sum_{j != i} W_ij.  W has a zero diagonal."""
    return np.asarray(W.sum(axis=1)).ravel()


def laplacian(g) -> sp.csr_matrix:
    """L = S - W."""
    W = adjacency(g)
    return (sp.diags(strengths(W)) - W).tocsr()


def laplacian_dense(g) -> np.ndarray:
    return laplacian(g).toarray()
