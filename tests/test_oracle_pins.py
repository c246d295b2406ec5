"""Pins of the fp64 oracle against things other than itself (task rule ③).

Every oracle function is checked against closed forms, invariants, brute force,
independent numerical methods or library routines -- never against a retyped
copy of its own formula.  CPU only.
"""

import itertools

import numpy as np
import pytest
import scipy.integrate
import scipy.sparse as sp
from numpy.polynomial import chebyshev as npcheb

import scinputs
from oracle import ari, chebyshev, eigencount, kmeans, lambda_max, laplacian, pipeline, stability

# ---------------------------------------------------------------------------
# §2.1 Laplacian  L = S - W
# ---------------------------------------------------------------------------


def test_laplacian_small_graphs_by_hand():
    # path 0-1-2: strengths (1,2,1); L 1 = 0
    L = laplacian.laplacian_dense(scinputs.path(3))
    assert np.allclose(np.diag(L), [1, 2, 1])
    assert np.allclose(L @ np.ones(3), 0)
    # triangle: L (1,-1,0) = (3,-3,0)? hand: L = 2I - (J - I) -> (2+1, -2-1, -1+1)
    L = laplacian.laplacian_dense(scinputs.complete(3))
    assert np.allclose(L @ np.array([1.0, -1.0, 0.0]), [3.0, -3.0, 0.0])
    # star K_{1,4}: centre strength 4, leaves 1
    L = laplacian.laplacian_dense(scinputs.star(4))
    assert np.allclose(np.diag(L), [4, 1, 1, 1, 1])


def test_laplacian_quadratic_form_brute_force():
    g = scinputs.random_connected(30, 0.2, seed=3)
    L = laplacian.laplacian(g)
    x = np.random.default_rng(0).standard_normal(g.n)
    # x^T L x = 1/2 sum_ij W_ij (x_i - x_j)^2 by an explicit loop over stored entries
    tot = 0.0
    for i in range(g.n):
        for e in range(g.row_ptr[i], g.row_ptr[i + 1]):
            j = g.col_idx[e]
            tot += 0.5 * float(g.values[e]) * (x[i] - x[j]) ** 2
    assert abs(x @ (L @ x) - tot) < 1e-10 * abs(tot)
    # symmetric, zero row sums, PSD
    Ld = L.toarray()
    assert np.array_equal(Ld, Ld.T)
    assert np.allclose(Ld.sum(axis=1), 0, atol=1e-12)
    assert np.linalg.eigvalsh(Ld)[0] > -1e-10


@pytest.mark.parametrize("n", [5, 8, 13])
def test_ring_and_path_closed_form_spectra(n):
    m = np.arange(n)
    lam_ring = np.sort(2 - 2 * np.cos(2 * np.pi * m / n))
    lam_path = np.sort(2 - 2 * np.cos(np.pi * m / n))
    assert np.allclose(np.linalg.eigvalsh(laplacian.laplacian_dense(scinputs.ring(n))), lam_ring)
    assert np.allclose(np.linalg.eigvalsh(laplacian.laplacian_dense(scinputs.path(n))), lam_path)
    # weighted ring scales the spectrum
    assert np.allclose(np.linalg.eigvalsh(laplacian.laplacian_dense(scinputs.ring(n, 2.5))),
                       2.5 * lam_ring, atol=1e-6)


# ---------------------------------------------------------------------------
# §4.1 step 1: lambda_N bound
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("g,exact", [
    (scinputs.path(3), 3.0),                       # dense 3x3: {0,1,3}
    (scinputs.complete(4), 4.0),                   # K_N: lambda_N = N
    (scinputs.from_edges(2, [0], [1], [0.7]), 1.4),  # single edge: 2w
    (scinputs.ring(10), 4.0),                      # even ring: 2 - 2cos(pi) = 4
])
def test_lambda_max_bound_closed_forms(g, exact):
    L = laplacian.laplacian(g)
    x0 = np.random.default_rng(1).standard_normal(g.n)
    b = lambda_max.lambda_max_bound(L, x0, iters=2000, margin=0.01)
    assert exact - 1e-6 <= b <= 1.02 * exact


def test_lambda_max_bound_random_graphs():
    for s in range(5):
        g = scinputs.random_connected(60, 0.1, seed=s)
        L = laplacian.laplacian(g)
        ex = np.linalg.eigvalsh(L.toarray())[-1]
        b = lambda_max.lambda_max_bound(L, np.random.default_rng(s).standard_normal(g.n), 3000, 0.01)
        assert ex <= b <= 1.05 * ex


# ---------------------------------------------------------------------------
# §2.3-2.4: Chebyshev coefficients, Jackson damping, the recurrence
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("ratio", [0.05, 0.3, 0.5, 0.77])
def test_coeffs_match_numerical_quadrature(ratio):
    """c_j = (2/pi) int_0^pi h(cos t) cos(j t) dt (j=0 halved), by adaptive quadrature."""
    lmax = 3.0
    lc = ratio * lmax
    c = chebyshev.lowpass_coeffs(lc, lmax, 12)
    a = 2 * lc / lmax - 1
    for j in range(13):
        f = lambda t: (1.0 if np.cos(t) <= a else 0.0) * np.cos(j * t)
        tc = np.arccos(a)
        val = scipy.integrate.quad(f, 0, tc, limit=200)[0] + scipy.integrate.quad(f, tc, np.pi, limit=200)[0]
        val *= 2 / np.pi
        if j == 0:
            val /= 2
        assert abs(c[j] - val) < 1e-9


def test_coeffs_special_cases():
    # all-pass: h == 1 on [0, lmax] -> c = (1, 0, 0, ...)
    c = chebyshev.lowpass_coeffs(5.0, 5.0, 20)
    assert abs(c[0] - 1) < 1e-15 and np.all(np.abs(c[1:]) < 1e-14)
    # all-stop
    c = chebyshev.lowpass_coeffs(0.0, 5.0, 20)
    assert np.all(np.abs(c) < 1e-14)
    # half cut: square-wave series of 1[x <= 0]: c0 = 1/2, even c_j = 0, c_1 = -2/pi, c_3 = +2/(3 pi)
    c = chebyshev.lowpass_coeffs(2.5, 5.0, 7)
    assert abs(c[0] - 0.5) < 1e-15
    assert np.allclose(c[2::2], 0, atol=1e-15)
    assert abs(c[1] + 2 / np.pi) < 1e-15 and abs(c[3] - 2 / (3 * np.pi)) < 1e-15


def test_partial_sums_converge_to_step():
    """Truncated series -> h pointwise away from the jump (Dirichlet), checked with
    numpy's independent Chebyshev evaluator."""
    c = chebyshev.lowpass_coeffs(1.0, 4.0, 4000)
    x = np.array([-0.95, -0.8, -0.6, 0.0, 0.5, 0.9])     # jump at a = -0.5
    v = npcheb.chebval(x, c)
    assert np.allclose(v, (x <= -0.5).astype(float), atol=2e-3)


def test_jackson_damping_properties():
    for p in [5, 20, 50, 200]:
        g = chebyshev.jackson(p)
        assert abs(g[0] - 1) < 1e-14
        assert abs(g[1] - np.cos(np.pi / (p + 2))) < 1e-14   # known first factor
        assert np.all(np.diff(g) < 0) and g[-1] > 0
        # Jackson kernel is positive: the damped step approximation stays in [0, 1]
        # and is (nearly) monotone (Gibbs overshoot removed); undamped overshoots.
        c = chebyshev.lowpass_coeffs(1.3, 4.0, p)
        x = np.linspace(-1, 1, 4001)
        vd = npcheb.chebval(x, c * g)
        assert vd.min() > -1e-12 and vd.max() < 1 + 1e-12
        assert np.diff(vd).max() < 1e-5        # monotone up to tiny end ripples
    vu = npcheb.chebval(np.linspace(-1, 1, 4001), chebyshev.lowpass_coeffs(1.3, 4.0, 50))
    assert vu.max() > 1.05


def _path_eigs(n):
    m = np.arange(n)
    lam = 2 - 2 * np.cos(np.pi * m / n)
    i = np.arange(n)
    V = np.cos(np.pi * np.outer(i + 0.5, m) / n)
    V[:, 0] *= np.sqrt(1.0 / n)
    V[:, 1:] *= np.sqrt(2.0 / n)
    return lam, V


def _cheb_filter_impl(impl, g, R, coeffs, lmax):
    """The two oracle implementations of the same definition: numpy (chebyshev.cheb_filter
    on L) and plain C with OpenMP rows (cfilter.cheb_filter on W's CSR)."""
    if impl == "numpy":
        return chebyshev.cheb_filter(laplacian.laplacian(g), R, coeffs, lmax)
    from oracle import cfilter
    return cfilter.cheb_filter(g, R, coeffs, lmax, nthreads=3)


@pytest.mark.parametrize("impl", ["numpy", "c"])
@pytest.mark.parametrize("damping", [False, True])
def test_filter_recurrence_vs_closed_form_path_eigenbasis(damping, impl):
    """F R = V diag(p(lambda)) V^T R with the DCT-II eigenbasis of the path graph
    (closed form) and p evaluated by numpy's chebval (independent of the recurrence)."""
    n, order = 40, 60
    lam, V = _path_eigs(n)
    assert np.allclose(V.T @ V, np.eye(n), atol=1e-12)
    lmax, lc = 4.0, 0.6
    coeffs = chebyshev.filter_coeffs(lc, lmax, order, damping)
    R = np.random.default_rng(5).standard_normal((n, 7))
    Y = _cheb_filter_impl(impl, scinputs.path(n), R, coeffs, lmax)
    pl = npcheb.chebval(2 * lam / lmax - 1, coeffs)
    Yex = V @ (pl[:, None] * (V.T @ R))
    assert np.linalg.norm(Y - Yex) <= 1e-11 * np.linalg.norm(Yex)


@pytest.mark.parametrize("impl", ["numpy", "c"])
def test_filter_recurrence_vs_dense_eig_random_weighted(impl):
    for s in range(4):
        g = scinputs.random_connected(50, 0.15, seed=10 + s)
        L = laplacian.laplacian(g)
        lam, chi = np.linalg.eigh(L.toarray())
        lmax = 1.01 * lam[-1]
        coeffs = chebyshev.filter_coeffs(0.3 * lmax, lmax, 45, s % 2 == 0)
        R = np.random.default_rng(s).standard_normal((g.n, 5))
        Y = _cheb_filter_impl(impl, g, R, coeffs, lmax)
        pl = npcheb.chebval(2 * lam / lmax - 1, coeffs)
        Yex = chi @ (pl[:, None] * (chi.T @ R))
        assert np.linalg.norm(Y - Yex) <= 1e-10 * np.linalg.norm(Yex)


def test_c_oracle_matches_numpy_oracle_and_constant_vector():
    """The C oracle against the numpy one (same definition, different summation order:
    agreement to rounding) on an unweighted SBM and a weighted kNN graph, plus the
    constant-vector identity F 1 = p(0) 1 (L 1 = 0) and thread-count independence."""
    from oracle import cfilter
    for g in (scinputs.sbm(800, 4, 12, 0.1, seed=3), scinputs.gmm_knn(600, 3, 4, 6, seed=2)):
        lmax = 2.0 * g.degrees().max() if g.values is None else 2.0 * np.max(
            np.add.reduceat(g.weights(), g.row_ptr[:-1]))
        coeffs = chebyshev.filter_coeffs(0.15 * lmax, lmax, 70, True)
        R = np.random.default_rng(1).standard_normal((g.n, 6))
        Yn = chebyshev.cheb_filter(laplacian.laplacian(g), R, coeffs, lmax)
        Yc = cfilter.cheb_filter(g, R, coeffs, lmax, nthreads=4)
        assert np.linalg.norm(Yc - Yn) <= 1e-12 * np.linalg.norm(Yn)
        assert np.array_equal(Yc, cfilter.cheb_filter(g, R, coeffs, lmax, nthreads=1))
        y1 = cfilter.cheb_filter(g, np.ones(g.n), coeffs, lmax)
        assert np.allclose(y1, npcheb.chebval(-1.0, coeffs), atol=1e-11)


def test_filter_approximates_ideal_projector_within_polynomial_error():
    """||F R - U_k U_k^T R|| <= max_l |p(lambda_l) - h(lambda_l)| ||R|| (F - H is diagonal
    in the eigenbasis), with U_k the closed-form first k path eigenvectors."""
    n, k, order = 20, 3, 300
    lam, V = _path_eigs(n)
    lmax = 4.0
    lc = 0.5 * (lam[k - 1] + lam[k])
    L = laplacian.laplacian(scinputs.path(n))
    coeffs = chebyshev.filter_coeffs(lc, lmax, order, True)
    R = np.random.default_rng(2).standard_normal((n, 16)) / 4.0
    Y = chebyshev.cheb_filter(L, R, coeffs, lmax)
    H = V[:, :k] @ (V[:, :k].T @ R)
    err_bound = np.max(np.abs(npcheb.chebval(2 * lam / lmax - 1, coeffs) - (lam <= lc)))
    assert err_bound < 0.1
    assert np.linalg.norm(Y - H, 2) <= err_bound * np.linalg.norm(R, 2) + 1e-12
    # the ideal-filter helper agrees with the closed form
    Hd = chebyshev.ideal_filter_dense(L.toarray(), R, lc)
    assert np.allclose(Hd, H, atol=1e-10)


def test_filter_constant_vector_and_linearity():
    g = scinputs.sbm(300, 3, 8, 0.1, seed=4)
    L = laplacian.laplacian(g)
    lmax = 2.0 * g.degrees().max()          # Gershgorin bound
    coeffs = chebyshev.filter_coeffs(0.2 * lmax, lmax, 40, True)
    one = np.ones((g.n, 1))
    # L 1 = 0  =>  T_j(L~) 1 = T_j(-1) 1 = (-1)^j 1  =>  F 1 = p(0) 1
    y = chebyshev.cheb_filter(L, one, coeffs, lmax)
    p0 = npcheb.chebval(-1.0, coeffs)
    assert np.allclose(y, p0, atol=1e-12)
    rng = np.random.default_rng(0)
    A, B = rng.standard_normal((g.n, 3)), rng.standard_normal((g.n, 3))
    lhs = chebyshev.cheb_filter(L, 2 * A - 3 * B, coeffs, lmax)
    rhs = 2 * chebyshev.cheb_filter(L, A, coeffs, lmax) - 3 * chebyshev.cheb_filter(L, B, coeffs, lmax)
    assert np.allclose(lhs, rhs, atol=1e-10)
    # symmetry <u, F v> = <F u, v>
    assert abs(np.sum(A * chebyshev.cheb_filter(L, B, coeffs, lmax))
               - np.sum(chebyshev.cheb_filter(L, A, coeffs, lmax) * B)) < 1e-9


def test_jl_expected_distance_equals_spectral_distance():
    """§3.1 Eq. (9): E ||f~_i - f~_j||^2 = ||f_i - f_j||^2 for R ~ N(0, 1/eta) with the
    ideal filter; the Monte-Carlo mean approaches it as the number of signals grows."""
    g = scinputs.two_cliques(8, 0.2)
    Ld = laplacian.laplacian_dense(g)
    lam, chi = np.linalg.eigh(Ld)
    k = 2
    U = chi[:, :k]
    lc = 0.5 * (lam[k - 1] + lam[k])
    D2 = np.sum((U[:, None, :] - U[None, :, :]) ** 2, axis=2)
    acc = np.zeros_like(D2)
    draws, eta = 400, 16
    for t in range(draws):
        R = scinputs.gaussian_block(t, g.n, eta).astype(np.float64)
        F = chebyshev.ideal_filter_dense(Ld, R, lc)
        acc += np.sum((F[:, None, :] - F[None, :, :]) ** 2, axis=2)
    acc /= draws
    mask = D2 > 1e-6
    rel = np.abs(acc[mask] - D2[mask]) / D2[mask]
    assert rel.max() < 0.1 and rel.mean() < 0.03


# ---------------------------------------------------------------------------
# §3.2 eigencount and dichotomy
# ---------------------------------------------------------------------------


def test_eigencount_exact_trace_ring():
    """With R = I (N unit probes) the estimator is exactly trace(F^2) = sum_l p(lambda_l)^2;
    for a mid-gap cut and high order it rounds to #{lambda_l <= lambda_c} (closed-form ring)."""
    n = 24
    lam = np.sort(2 - 2 * np.cos(2 * np.pi * np.arange(n) / n))
    L = laplacian.laplacian(scinputs.ring(n))
    for kk in [1, 3, 5, 9]:
        lc = 0.5 * (lam[kk - 1] + lam[kk])
        cnt = eigencount.count_below(L, lc, 4.0, 250, np.eye(n), damping=True)
        pl = npcheb.chebval(2 * lam / 4.0 - 1, chebyshev.filter_coeffs(lc, 4.0, 250, True))
        assert abs(cnt - np.sum(pl ** 2)) < 1e-9
        assert round(cnt) == kk


def test_eigencount_hutchinson_random_probes():
    n = 24
    lam = np.sort(2 - 2 * np.cos(2 * np.pi * np.arange(n) / n))
    L = laplacian.laplacian(scinputs.ring(n))
    lc = 0.5 * (lam[4] + lam[5])
    R = scinputs.gaussian_block(11, n, 400).astype(np.float64)
    cnt = eigencount.count_below(L, lc, 4.0, 250, R, True)
    assert abs(cnt - 5) < 1.0


def test_dichotomy_lands_in_kth_gap_path():
    n = 20
    lam, _ = _path_eigs(n)
    L = laplacian.laplacian(scinputs.path(n))
    for k in [1, 3, 6]:
        lk, ck, trace = eigencount.estimate_lambda_k(L, k, 4.0, 300, np.eye(n), True, 40, 1e-4)
        width = 4.0 * np.pi / 300         # transition half-width of the damped step
        assert lam[k - 1] - width <= lk < lam[k]
        assert ck >= k - 0.5
        # bracket invariant along the trace
        assert all((c >= k - 0.5) == (m >= lk) for m, c in trace if m == lk or c < k - 0.5)


# ---------------------------------------------------------------------------
# k-means, ARI, stability
# ---------------------------------------------------------------------------


def _blobs(seed, n_per=40, k=4, dim=5, spread=0.3):
    rng = np.random.default_rng(seed)
    centers = rng.uniform(-5, 5, size=(k, dim))
    X = np.concatenate([c + spread * rng.standard_normal((n_per, dim)) for c in centers])
    return X.astype(np.float32)


def test_kmeans_lloyd_matches_sklearn():
    from sklearn.cluster import KMeans
    for s in range(5):
        X = _blobs(s)
        k = 4
        u = scinputs.uniforms(s, k)
        seeds = kmeans.kmeanspp(X, k, u)
        C0 = X[seeds].astype(np.float64)
        lab, C, inertia, it = kmeans.lloyd(X, C0, 100)
        sk = KMeans(n_clusters=k, init=C0, n_init=1, max_iter=100, tol=0.0, algorithm="lloyd").fit(X.astype(np.float64))
        assert np.array_equal(lab, sk.labels_)
        assert np.allclose(C, sk.cluster_centers_, atol=1e-10)
        assert abs(inertia - sk.inertia_) < 1e-8 * max(1.0, inertia)


def test_kmeans_brute_force_and_degenerate():
    # 4 corners of a long rectangle, k=2: optimum over all 7 bipartitions
    X = np.array([[0, 0], [0, 1], [10, 0], [10, 1]], dtype=np.float32)
    best = min(
        sum(np.sum((X[list(S)] - X[list(S)].mean(0)) ** 2) for S in (A, tuple(set(range(4)) - set(A))))
        for r in (1, 2) for A in itertools.combinations(range(4), r))
    lab, C, inertia, _ = kmeans.lloyd(X, X[[0, 2]].astype(np.float64), 50)
    assert abs(inertia - best) < 1e-12 and lab[0] == lab[1] != lab[2] == lab[3]
    # k = 1: inertia = total squared deviation
    Xr = _blobs(3)
    lab, C, inertia, _ = kmeans.lloyd(Xr, Xr[:1].astype(np.float64), 10)
    Xd = Xr.astype(np.float64)
    assert np.all(lab == 0) and abs(inertia - np.sum((Xd - Xd.mean(0)) ** 2)) < 1e-8
    # k = N: inertia 0
    lab, C, inertia, _ = kmeans.lloyd(X, X.astype(np.float64), 10)
    assert inertia == 0.0 and len(set(lab)) == 4


def test_kmeanspp_hand_example():
    X = np.array([[0.0], [1.0], [10.0]])
    # u0 = 0 -> index 0; D^2 = (0, 1, 100), cumsum (0, 1, 101)
    assert list(kmeans.kmeanspp(X, 2, np.array([0.0, 0.5]))) == [0, 2]     # 50.5 -> idx 2
    assert list(kmeans.kmeanspp(X, 2, np.array([0.0, 0.005]))) == [0, 1]   # 0.505 -> idx 1
    assert list(kmeans.kmeanspp(X, 2, np.array([0.99, 0.0]))) == [2, 0]    # D^2 = (100, 81, 0)


def test_kmeans_best_replicate_rule_hand_example():
    """Replicate selection (oracle/kmeans.py kmeans(): lowest inertia wins, ties -> lowest
    replicate index; R8, §5 l.404 'replicates').  1-D points
    A = {0, 1}, B = {10, 11}, C = {100, 120}, k = 3, four restarts whose seeds (chosen by
    hand through the D^2 cumulative sums) converge to two different local optima:
      r0, r3: seeds 0, 10, 100 -> {A}, {B}, {C}:   inertia 4 * 0.25 + 2 * 100   = 201
      r1:     seeds 100, 120, 0 -> {100}, {120}, {A u B}: 2 * 5.5^2 + 2 * 4.5^2 = 101
      r2:     seeds 120, 100, 1 -> {120}, {100}, {A u B}: 101 (an exact tie with r1,
              different label numbering)
    Expected: replicate 1 (not 2: ties go to the lowest index; not 0 or 3: the minimum)."""
    X = np.array([[0.0], [1.0], [10.0], [11.0], [100.0], [120.0]])
    u = np.array([[0.0, 0.002, 0.2],      # seeds 0, 2, 4 (hand cumsums in the docstring)
                  [0.7, 0.995, 0.1],      # seeds 4, 5, 0
                  [0.9, 0.995, 0.4],      # seeds 5, 4, 1
                  [0.0, 0.002, 0.2]])
    assert list(kmeans.kmeanspp(X, 3, u[0])) == [0, 2, 4]
    assert list(kmeans.kmeanspp(X, 3, u[1])) == [4, 5, 0]
    assert list(kmeans.kmeanspp(X, 3, u[2])) == [5, 4, 1]
    labels, C, inertia, it, r, seeds = kmeans.kmeans(X, 3, u, 50)
    assert r == 1 and inertia == 101.0
    assert list(labels) == [2, 2, 2, 2, 0, 1]
    assert np.array_equal(C[:, 0], [100.0, 120.0, 5.5])
    # the single-restart results the rule chooses among
    assert kmeans.kmeans(X, 3, u[:1], 50)[2] == 201.0
    assert list(kmeans.kmeans(X, 3, u[2:3], 50)[0]) == [2, 2, 2, 2, 1, 0]
    # order matters only through the index: the tie goes to whichever comes first
    assert kmeans.kmeans(X, 3, u[[2, 1]], 50)[4] == 0
    assert list(kmeans.kmeans(X, 3, u[[0, 3]], 50)[0]) == [0, 0, 1, 1, 2, 2]


def test_poly_eval_against_chebval_and_hand_values():
    """oracle/chebyshev.py poly_eval: p(lambda) = sum_j c_j T_j(x), x = 2 lambda / lambda_max - 1
    (R1).  Pinned to hand values of T_0..T_3 and to numpy's Clenshaw evaluation
    (numpy.polynomial.chebyshev.chebval), an independent routine."""
    lmax = 4.0
    # x = -1, -0.5, 0, 0.5, 1 at lambda = 0, 1, 2, 3, 4
    lam = np.array([0.0, 1.0, 2.0, 3.0, 4.0])
    assert np.allclose(chebyshev.poly_eval(lam, np.array([1.0]), lmax), 1.0)
    assert np.allclose(chebyshev.poly_eval(lam, np.array([0.0, 1.0]), lmax), [-1, -0.5, 0, 0.5, 1])
    assert np.allclose(chebyshev.poly_eval(lam, np.array([0.0, 0.0, 1.0]), lmax), [1, -0.5, -1, -0.5, 1])
    assert np.allclose(chebyshev.poly_eval(lam, np.array([0.0, 0.0, 0.0, 1.0]), lmax), [-1, 1, 0, -1, 1])
    rng = np.random.default_rng(5)
    for p in (1, 7, 50, 300):
        c = rng.standard_normal(p + 1)
        lam = rng.uniform(0.0, lmax, 64)
        want = npcheb.chebval(2.0 * lam / lmax - 1.0, c)
        assert np.allclose(chebyshev.poly_eval(lam, c, lmax), want, rtol=1e-10, atol=1e-10 * np.abs(c).sum())
    # the filter's polynomial at 0 (the value F 1 = p(0) 1 uses) for the damped step
    d = chebyshev.filter_coeffs(0.3, 4.0, 40, True)
    assert chebyshev.poly_eval(0.0, d, 4.0) == pytest.approx(npcheb.chebval(-1.0, d), rel=1e-12)


def _recurrence_error(ratio, m, damping, theta=0.1, n_grid=10000):
    """|h - p_m| on the order grid with p_m evaluated a second way: the three-term
    recurrence of cheb_filter (pinned above on closed-form spectra) applied to the diagonal
    matrix diag(grid), i.e. the filter's own route, not the trigonometric form."""
    lam = chebyshev.order_grid(ratio, theta, n_grid)
    D = sp.diags(lam).tocsr()
    p = chebyshev.cheb_filter(D, np.ones((lam.size, 1)), chebyshev.filter_coeffs(ratio, 1.0, m, damping),
                              1.0)[:, 0]
    return np.max(np.abs((lam <= ratio).astype(float) - p))


def test_minimal_order_special_cases_and_monotone():
    """oracle/chebyshev.py minimal_order (§2.4 Eq. (4) l.151-162, reading R18).
    ratio = 1: h = 1 on [0, 1], c = (1, 0, ...), so m* = 1 with zero error (damped or not);
    sharper cuts need higher orders (m* non-increasing in the ratio on a decade grid; PAPER.md
    §5 l.407-409: small lambda_k/lambda_N "necessitates a large m"); Jackson damping widens the
    transition, so it never needs a lower order than the undamped series at these ratios; a
    stricter delta never needs a lower order."""
    for damping in (False, True):
        assert chebyshev.minimal_order(1.0, 0.1, damping, 10) == 1
        assert chebyshev.approx_error(1.0, 1, damping) == pytest.approx(0.0, abs=1e-15)
    ms = [chebyshev.minimal_order(r, 0.1, False, 300) for r in (1e-2, 3e-2, 1e-1, 0.5)]
    assert all(a > b for a, b in zip(ms, ms[1:])), ms
    msd = [chebyshev.minimal_order(r, 0.1, True, 300) for r in (1e-1, 0.3, 0.5)]
    assert all(a > b for a, b in zip(msd, msd[1:])), msd
    assert msd[0] >= ms[2] and msd[2] >= ms[3]
    assert chebyshev.minimal_order(0.1, 0.05, False, 300) >= ms[2]


@pytest.mark.parametrize("ratio,damping", [(0.5, False), (0.1, False), (0.03, True), (0.3, True)])
def test_minimal_order_against_recurrence_route(ratio, damping):
    """The error approx_error measures equals the one of the recurrence route, and m* is
    minimal under that route: m* meets delta, m* - 1 does not (a wrong band, coefficient or
    damping flag in either route fails this)."""
    m = chebyshev.minimal_order(ratio, 0.1, damping, 400)
    assert m is not None and m >= 2
    for mm in (m - 1, m, m + 3):
        assert chebyshev.approx_error(ratio, mm, damping) == pytest.approx(
            _recurrence_error(ratio, mm, damping), abs=1e-9)
    assert _recurrence_error(ratio, m, damping) <= 0.1
    assert _recurrence_error(ratio, m - 1, damping) > 0.1


def test_minimal_order_band_is_required():
    """Without the transition band (theta = 0) and with lambda_c on the grid, h jumps between
    grid points 1/(n_grid-1) apart, and a continuous polynomial of moderate order cannot stay
    within 0.1 of both sides (its value at the cut and the neighbour differ by < 0.8 for
    m <= 300): no order is found -- the reason for reading R18."""
    assert chebyshev.minimal_order(0.5, 0.1, False, 300, theta=0.0, n_grid=10001) is None
    assert chebyshev.minimal_order(0.5, 0.1, False, 300, theta=0.1, n_grid=10001) is not None


def test_kmeans_inertia_monotone():
    X = _blobs(7, spread=2.0).astype(np.float64)
    C = X[:4].copy()
    lab, _ = kmeans.assign(X, C)
    prev = np.inf
    for _ in range(20):
        C = kmeans.update(X, lab, C)
        lab, d = kmeans.assign(X, C)
        assert d.sum() <= prev + 1e-9
        prev = d.sum()


def test_ari_against_sklearn_and_hand_cases():
    from sklearn.metrics import adjusted_rand_score
    assert ari.ari([0, 0, 1, 1], [0, 1, 0, 1]) == pytest.approx(-0.5)
    assert ari.ari([0, 0, 1, 1, 2], [5, 5, 7, 7, 1]) == 1.0
    rng = np.random.default_rng(0)
    for _ in range(20):
        a = rng.integers(0, 5, 200)
        b = rng.integers(0, 7, 200)
        assert ari.ari(a, b) == pytest.approx(adjusted_rand_score(a, b), abs=1e-12)
        assert ari.ari(a, b) == ari.ari(b, a)
        perm = rng.permutation(7)
        assert ari.ari(a, perm[b]) == pytest.approx(ari.ari(a, b), abs=1e-15)
    # chance level
    vals = [ari.ari(rng.integers(0, 10, 1000), rng.integers(0, 10, 1000)) for _ in range(50)]
    assert abs(np.mean(vals)) < 0.01
    # degenerate: both single-cluster
    assert ari.ari([0, 0, 0], [1, 1, 1]) == 1.0


def test_stability_gamma():
    a, b, c = [0, 0, 1, 1], [0, 1, 0, 1], [1, 1, 0, 0]
    assert stability.gamma([a, b]) == pytest.approx(-0.5)
    assert stability.gamma([a, c]) == 1.0
    assert stability.gamma([a, b, c]) == pytest.approx((-0.5 + 1.0 - 0.5) / 3)
    assert stability.k_star({2: 0.9, 3: 0.95, 4: 0.95}) == 3


# ---------------------------------------------------------------------------
# whole pipeline on a trivially separable instance
# ---------------------------------------------------------------------------


def test_pipeline_recovers_planted_sbm():
    g = scinputs.sbm(600, 3, 12, 0.02, seed=8)
    R = scinputs.gaussian_block(1, g.n, 12).astype(np.float64)
    Rp = scinputs.gaussian_block(2, g.n, 20, stream=2).astype(np.float64)
    u = np.stack([scinputs.uniforms(3, 3, offset=3 * r) for r in range(5)])
    L = laplacian.laplacian(g)
    lm = lambda_max.lambda_max_exact(L) * 1.01
    out = pipeline.accelerated_sc(g, 3, R, Rp, 80, True, u, lambda_max_value=lm)
    assert ari.ari(out["labels"], g.labels) > 0.95
    assert out["count_k"] >= 2.5


def test_normalize_rows():
    F = np.array([[3.0, 4.0], [0.0, 0.0], [1.0, 0.0]])
    N = pipeline.normalize_rows(F)
    assert np.allclose(N, [[0.6, 0.8], [0, 0], [1, 0]])
