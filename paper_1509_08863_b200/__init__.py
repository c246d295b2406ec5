"""B200-native accelerated spectral clustering (arXiv:1509.08863) -- hot path.

The product is the C-ABI library ``libsc_b200.so`` (include/sc_b200.h); this
package is its thin Python binding (``_lib``: one function per C entry point,
argument marshalling only) plus a small ``Graph`` handle wrapper and the
row-partitioned multi-GPU driver (``dist``).  Importing the package fails
loudly when the library is missing: there is no CPU fallback.
"""

from __future__ import annotations

from . import _lib
from ._lib import *  # noqa: F401,F403  (sc_* functions)
from ._lib import SCError


class Graph:
    """Owns an ``sc_graph`` handle (device-resident CSR of W + strengths)."""

    def __init__(self, n_rows, row_ptr, col_idx, values=None, n_cols=None):
        self.n_rows = int(n_rows)
        self.n_cols = int(n_cols if n_cols is not None else n_rows)
        self.nnz = int(row_ptr[-1])
        self.handle = _lib.sc_graph_load(self.n_rows, self.n_cols, self.nnz, row_ptr, col_idx, values)

    @classmethod
    def from_csr(cls, g):
        """From an object with n, row_ptr, col_idx, values (e.g. scinputs.CSRGraph)."""
        return cls(g.n, g.row_ptr, g.col_idx, g.values)

    def info(self):
        return _lib.sc_graph_info(self.handle)

    def close(self):
        if getattr(self, "handle", None):
            _lib.sc_graph_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


__all__ = ["Graph", "SCError"] + _lib.EXPORTED
