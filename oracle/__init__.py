"""ORACLE -- TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct fp64 CPU implementation of what the
accelerated spectral clustering hot path computes (PAPER.md = arxiv 1509.08863,
"Accelerated spectral clustering using graph filtering of random signals").

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import or execute anything in
this package.  The product path (``paper_1509_08863_b200``) never imports it,
and this package never imports the product path: the two share no code.  The
only shared module is ``scinputs`` (seeded input generators, none of the
method's arithmetic).

Modules (each function cites the PAPER.md passage it follows):
    laplacian   -- L = S - W                                   (§2.1)
    lambda_max  -- power-iteration estimate of lambda_N         (§4.1 step 1)
    chebyshev   -- ideal low-pass h_{lambda_c}, Chebyshev coefficients,
                   Jackson damping, fast filtering F^m_h R     (§2.3, §2.4, §3.2)
    eigencount  -- eigenvalue count below lambda_c, dichotomy   (§3.2)
    kmeans      -- k-means++ seeding + Lloyd iterations         (§2.2 step 4, §4.1 step 6)
    ari         -- adjusted Rand index                          (§4.3, §5)
    stability   -- gamma(k), Eq. (11)                           (§4.3)
    pipeline    -- the six-step accelerated algorithm           (§4.1)
    cfilter     -- chebyshev.cheb_filter written out in plain C, rows of each step on
                   OpenMP threads (full-size columns, all-core cpu_baseline)   (§2.4, §4.1)

Parity status of every function is recorded in DESIGN.md §"Oracle pins".
"""

from . import laplacian, lambda_max, chebyshev, eigencount, kmeans, ari, stability, pipeline  # noqa: F401
