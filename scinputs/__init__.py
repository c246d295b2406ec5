"""Seeded synthetic inputs shared by the oracle, the tests and bench.py.

This package holds NO arithmetic of the paper's method (no Laplacian, no
Chebyshev filter, no k-means).  It only builds the inputs the method consumes:

* ``graphs``  -- symmetric CSR similarity graphs W (SBM, Gaussian-mixture kNN,
  Chung-Lu power-law degrees, ring / path / complete / star / two-clique fixtures,
  RCM relabelling).  Graph construction is
  step 1 of PAPER.md §2.2 / §4.1 ("compute the pairwise similarities s_ij,
  create a similarity graph W"), which the paper leaves unchanged.
* ``signals`` -- a counter-based Gaussian generator for the random signal
  block R (§3.1, §4.1 step 4 line 316: i.i.d. Gaussian,
  mean 0, variance 1/eta) and uniforms for k-means++ draws.  The CUDA library
  implements the same counter-based generator on device (``sc_random_signals``)
  so both sides see the same numbers.
* ``configs`` -- the five BASELINE.json workloads as builders.

Both ``oracle/`` and ``paper_1509_08863_b200`` may import this package; it
imports neither of them.
"""

from .graphs import (CSRGraph, sbm, gmm_knn, ring, path, complete, star, two_cliques, from_edges, random_connected,
                     chung_lu, permute, rcm_order)
from .signals import gaussian_block, uniforms, splitmix64

__all__ = [
    "CSRGraph", "sbm", "gmm_knn", "ring", "path", "complete", "star", "two_cliques",
    "from_edges", "random_connected", "chung_lu", "permute", "rcm_order", "gaussian_block", "uniforms", "splitmix64",
]
