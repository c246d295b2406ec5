"""CPU-side checks of the native library: it loads, exports every symbol the
header declares, its host-only math agrees with the oracle, and compute calls
fail loudly (no CPU fallback) when there is no GPU."""

import ctypes
import os
import re

import numpy as np
import pytest
from numpy.polynomial import chebyshev as npcheb

import scinputs
from oracle import chebyshev, eigencount, laplacian

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sc_b200.h")


@pytest.fixture(scope="module")
def sc():
    import native_build
    native_build.build()
    import paper_1509_08863_b200 as sc
    return sc


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(sc_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol(sc):
    lib = ctypes.CDLL(sc._lib.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # the binding wraps every declared entry point under the same name
    assert set(syms) <= set(sc._lib.EXPORTED)


def test_host_coefficients_match_oracle(sc):
    for lc, lm, p, jk in [(1.0, 4.0, 5, True), (0.3, 25.0, 300, False), (2.0, 4.0, 50, True), (4.0, 4.0, 7, False)]:
        c = sc.sc_cheby_coeffs(lc, lm, p, jk)
        o = chebyshev.filter_coeffs(lc, lm, p, jk)
        assert np.allclose(c, o, rtol=1e-13, atol=1e-15)


def _ring_moments(n):
    """mu_m = trace T_m(L~) = sum_l T_m(x_l) for R = I on the ring (closed-form spectrum)."""
    lam = 2 - 2 * np.cos(2 * np.pi * np.arange(n) / n)
    x = 2 * lam / 4.0 - 1
    return lambda order: np.array([npcheb.chebval(x, np.eye(2 * order + 1)[m]).sum() for m in range(2 * order + 1)])


def test_host_eigencount_from_moments_matches_oracle(sc):
    n, order = 24, 120
    mu = _ring_moments(n)(order)
    L = laplacian.laplacian(scinputs.ring(n))
    for lc in [0.05, 0.4, 1.3, 2.9]:
        c = sc.sc_eigencount_from_moments(mu, order, lc, 4.0, True)
        o = eigencount.count_below(L, lc, 4.0, order, np.eye(n), True)
        assert abs(c - o) < 1e-9 * n


def test_host_dichotomy_matches_oracle(sc):
    n, order = 24, 150
    mu = _ring_moments(n)(order)
    L = laplacian.laplacian(scinputs.ring(n))
    for k in [1, 3, 5, 9]:
        lk, ck = sc.sc_lambda_k_from_moments(mu, order, k, 4.0, True, 30, 1e-3)
        lo, co, _ = eigencount.estimate_lambda_k(L, k, 4.0, order, np.eye(n), True, 30, 1e-3)
        assert lk == lo and abs(ck - co) < 1e-9 * n


def test_compute_calls_fail_loudly_without_gpu(sc):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    g = scinputs.path(5)
    with pytest.raises(sc.SCError):
        sc.sc_graph_load(g.n, g.n, g.nnz, g.row_ptr, g.col_idx, g.values)
    with pytest.raises(sc.SCError):
        sc.sc_random_signals_f32(4, 2, 0, 1, 0, 0.0, np.zeros((4, 2), np.float32))


def test_argument_errors(sc):
    with pytest.raises(sc.SCError):
        sc.sc_cheby_coeffs(1.0, -1.0, 5, False)
    with pytest.raises(sc.SCError):
        sc.sc_lambda_k_from_moments(np.zeros(11), 5, 0, 4.0, True)
    # sc_filter_order: ratio outside (0, 1], delta <= 0, theta outside [0, 1), n_grid < 2, m_max outside [1, 4096]
    for bad in [dict(ratio=0.0), dict(ratio=1.5), dict(delta=0.0), dict(theta=-0.1), dict(theta=1.0),
                dict(n_grid=1), dict(m_max=0), dict(m_max=5000)]:
        kw = dict(ratio=0.1, delta=0.1, jackson=False, theta=0.1, n_grid=100, m_max=10)
        kw.update(bad)
        with pytest.raises(sc.SCError):
            sc.sc_filter_order(**kw)


def test_argument_errors_new_entry_points(sc):
    """Argument checks run before any device work (no GPU needed)."""
    import ctypes
    lib = sc._lib._lib
    gamma = np.zeros(3)
    # null graph / bad k range / J < 2
    assert lib.sc_stability(None, 2, 4, 3, 8, 10, 1, 4, ctypes.c_uint64(1), 1, 10, ctypes.c_double(0.0), None,
                            gamma.ctypes.data, None, None, None) == -1
    assert lib.sc_dist_create(None, None, 0, None, 0, None, None, None) == -1
    out = ctypes.c_void_p()
    uid = ctypes.create_string_buffer(128)
    assert lib.sc_comm_init(uid, 0, 0, ctypes.byref(out)) == -1      # world < 1
    assert lib.sc_comm_init(uid, 2, 2, ctypes.byref(out)) == -1      # rank >= world
    assert lib.sc_nccl_unique_id(None) == -1
    assert lib.sc_dist_filter_f32(None, None, 1, ctypes.c_double(1.0), 4, None, None, None) == -1
    assert "argument" in sc.sc_last_error() or "null" in sc.sc_last_error()
    with pytest.raises(sc.SCError):
        sc.sc_kmeans(np.zeros((4, 2), np.float32), 4, 2, 5, 1, 10, 0, None, np.zeros(4, np.int32))   # k > n
