"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle.

Tolerances (BASELINE.json north_star): filtered block relative Frobenius error
<= 1e-4 in fp32 and <= 1e-10 in fp64; k-means labels bit-exact from shared
seeding; integer work (contingency tables, labels) exact.
"""

import os

import numpy as np
import pytest

import dist_reference as dref
import scinputs
from oracle import ari as oari
from oracle import chebyshev, eigencount, kmeans, lambda_max, laplacian, pipeline

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

F32_TOL = 1e-4
F64_TOL = 1e-10


@pytest.fixture(scope="module")
def sc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1509_08863_b200 as sc
    return sc


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-300))


def gpu_filter(sc, g, X, lc, lmax, order, jackson, dtype=torch.float32, G=None):
    own = G is None
    G = G or sc.Graph.from_csr(g)
    Xd = torch.from_numpy(np.ascontiguousarray(X)).to(dtype).cuda()
    Yd = torch.empty_like(Xd)
    f = sc.sc_filter_lowpass_f32 if dtype == torch.float32 else sc.sc_filter_lowpass_f64
    f(G.handle, lc, lmax, order, jackson, X.shape[1], 0, Xd, Yd)
    torch.cuda.synchronize()
    if own:
        G.close()
    return Yd.cpu().numpy()


# ---------------------------------------------------------------------------
# random signals (counter-based generator shared by definition)
# ---------------------------------------------------------------------------

def test_random_signals_match_host_generator(sc):
    for n, R, row0, seed in [(1000, 32, 0, 1), (777, 5, 123, 99), (4096, 24, 0, 2 ** 63 + 5)]:
        out = torch.empty((n, R), dtype=torch.float32, device="cuda")
        sc.sc_random_signals_f32(n, R, row0, seed, 0, 0.0, out)
        ref = scinputs.gaussian_block(seed, n, R, row0=row0)
        got = out.cpu().numpy()
        diff = got != ref
        assert diff.mean() < 1e-5
        assert np.all(np.abs(got - ref) <= np.spacing(np.abs(ref)) * 1.0001)
        out64 = torch.empty((n, R), dtype=torch.float64, device="cuda")
        sc.sc_random_signals_f64(n, R, row0, seed, 2, 0.5, out64)
        ref64 = scinputs.gaussian_block(seed, n, R, row0=row0, dtype=np.float64, variance=0.5, stream=2)
        assert np.allclose(out64.cpu().numpy(), ref64, rtol=1e-14, atol=1e-15)


# ---------------------------------------------------------------------------
# graph load, strengths, lambda_max
# ---------------------------------------------------------------------------

def test_strengths_match_oracle(sc):
    for g in [scinputs.random_connected(300, 0.05, seed=1), scinputs.sbm(2000, 5, 10, 0.1, seed=3),
              scinputs.gmm_knn(3000, 5, 4, 8, seed=2)]:
        G = sc.Graph.from_csr(g)
        s = np.empty(g.n, dtype=np.float64)
        sc.sc_graph_strengths(G.handle, s)
        so = laplacian.strengths(laplacian.adjacency(g))
        assert np.allclose(s, so, rtol=1e-13, atol=0)
        n_rows, n_cols, nnz, smax = G.info()
        assert (n_rows, n_cols, nnz) == (g.n, g.n, g.nnz) and smax == pytest.approx(so.max(), rel=1e-13)


def test_graph_load_rejects_bad_csr(sc):
    g = scinputs.path(5)
    bad = g.col_idx.copy()
    bad[0] = 7
    with pytest.raises(sc.SCError):
        sc.sc_graph_load(g.n, g.n, g.nnz, g.row_ptr, bad, None)
    with pytest.raises(sc.SCError):
        sc.sc_graph_load(g.n, g.n, g.nnz + 1, g.row_ptr, g.col_idx, None)
    shifted = g.row_ptr + 1
    with pytest.raises(sc.SCError):
        sc.sc_graph_load(g.n, g.n, g.nnz + 1, shifted, np.concatenate([g.col_idx, [0]]).astype(np.int32), None)


@pytest.mark.parametrize("maker", [
    lambda: scinputs.sbm(2000, 5, 10, 0.1, seed=1234),
    lambda: scinputs.gmm_knn(5000, 10, 10, 10, seed=5),
    lambda: scinputs.ring(101),
    lambda: scinputs.complete(30),
])
def test_lambda_max_is_a_tight_upper_bound(sc, maker):
    g = maker()
    G = sc.Graph.from_csr(g)
    b = sc.sc_lambda_max(G.handle, 80, 0.01, 11)
    L = laplacian.laplacian(g)
    if g.n <= 3000:
        ex = lambda_max.lambda_max_exact(L)
    else:
        import scipy.sparse.linalg as sla
        ex = float(sla.eigsh(L, k=1, which="LA", return_eigenvectors=False, tol=1e-10)[0])
    assert ex * (1 - 1e-9) <= b <= 1.02 * ex


# ---------------------------------------------------------------------------
# the fused Chebyshev filter
# ---------------------------------------------------------------------------

CASES = [
    # (graph maker, R, order, jackson, ratio lambda_c / lambda_max)
    ("c0_sbm", lambda: scinputs.sbm(2000, 5, 10, 0.1, seed=1234), 32, 50, True, 0.08),
    ("gmm_knn_w", lambda: scinputs.gmm_knn(4000, 10, 10, 10, seed=7), 24, 100, False, 0.01),
    ("er_weighted", lambda: scinputs.random_connected(500, 0.02, seed=9), 16, 30, True, 0.3),
    ("ragged_R5", lambda: scinputs.sbm(1531, 3, 9, 0.1, seed=4), 5, 20, False, 0.2),
    ("R1", lambda: scinputs.sbm(600, 3, 9, 0.1, seed=5), 1, 17, True, 0.2),
    ("R3_order1", lambda: scinputs.random_connected(97, 0.1, seed=6), 3, 1, False, 0.5),
    ("order2", lambda: scinputs.random_connected(97, 0.1, seed=6), 8, 2, False, 0.5),
    ("order3", lambda: scinputs.random_connected(97, 0.1, seed=6), 8, 3, True, 0.5),
    ("wide_R96", lambda: scinputs.sbm(3000, 6, 12, 0.1, seed=8), 96, 40, False, 0.1),
    ("wide_R200", lambda: scinputs.sbm(1200, 4, 12, 0.1, seed=8), 200, 12, True, 0.1),
    ("star_hub", lambda: scinputs.star(700), 8, 25, False, 0.3),
    # a 40 000-degree hub: its tile's column segment exceeds the staged capacity (the
    # streaming kernel reads it from global memory) and the resident plan does not fit
    ("hub_overflow", lambda: scinputs.from_edges(
        40001, np.concatenate([np.zeros(40000, np.int64), np.arange(1, 40000)]),
        np.concatenate([np.arange(1, 40001), np.arange(2, 40001)]), None), 16, 12, False, 0.3),
    ("path_tiny", lambda: scinputs.path(2), 4, 5, False, 0.5),
    # power-law degrees (Chung-Lu, exponent 2.1): hundreds of rows above the split threshold
    ("chung_lu", lambda: scinputs.chung_lu(30000, 20, 2.1, seed=3), 16, 30, True, 0.1),
]

# streaming paths: "streaming" = the SELL kernel (large graphs' default; rows above the split
# threshold of 128 go through hub_chunk_kernel), "split" = SELL with every row of degree > 4
# split, "csr" = the plain-CSR step kernel (SC_SELL=0; moments and partitioned paths),
# "halves" = the split gather
PATHS = {"resident": {"SC_RESIDENT": "1"}, "streaming": {"SC_RESIDENT": "0"},
         "split": {"SC_RESIDENT": "0", "SC_SELL_HUB_DEG": "4"}, "csr": {"SC_RESIDENT": "0", "SC_SELL": "0"},
         # split gather: the columns in two halves, two launches per step (SC_SELL_SPLIT=2 forces
         # it on small graphs; configs[3] takes it by default), with a sigma window of 256 rows
         "halves": {"SC_RESIDENT": "0", "SC_SELL_SPLIT": "2", "SC_SELL_SIGMA": "256", "SC_SELL_HUB_DEG": "64"}}


def _path_env(monkeypatch, path):
    for k, v in PATHS[path].items():
        monkeypatch.setenv(k, v)


@pytest.mark.parametrize("path", list(PATHS))
@pytest.mark.parametrize("name,maker,R,order,jackson,ratio", CASES, ids=[c[0] for c in CASES])
def test_filter_f32_parity(sc, name, maker, R, order, jackson, ratio, path, monkeypatch):
    # small graphs take the resident-CSR cooperative kernel by default; SC_RESIDENT=0 forces
    # the streaming per-step kernels on the same inputs
    _path_env(monkeypatch, path)
    g = maker()
    L = laplacian.laplacian(g)
    lmax = 2.0 * float(laplacian.strengths(laplacian.adjacency(g)).max())
    X = scinputs.gaussian_block(17, g.n, R)
    Y = gpu_filter(sc, g, X, ratio * lmax, lmax, order, jackson)
    Yo = chebyshev.lowpass_filter(L, X.astype(np.float64), ratio * lmax, lmax, order, jackson)
    assert rel(Y, Yo) <= F32_TOL


F64_CASES = CASES[:6] + [c for c in CASES if c[0] in ("star_hub", "chung_lu")]


@pytest.mark.parametrize("path", list(PATHS))
@pytest.mark.parametrize("name,maker,R,order,jackson,ratio", F64_CASES, ids=[c[0] for c in F64_CASES])
def test_filter_f64_parity(sc, name, maker, R, order, jackson, ratio, path, monkeypatch):
    _path_env(monkeypatch, path)
    g = maker()
    L = laplacian.laplacian(g)
    lmax = 2.0 * float(laplacian.strengths(laplacian.adjacency(g)).max())
    X = scinputs.gaussian_block(17, g.n, R, dtype=np.float64)
    Y = gpu_filter(sc, g, X, ratio * lmax, lmax, order, jackson, dtype=torch.float64)
    Yo = chebyshev.lowpass_filter(L, X, ratio * lmax, lmax, order, jackson)
    assert rel(Y, Yo) <= F64_TOL


@pytest.mark.parametrize("chunk", ["4", "8", "16", "32"])
def test_filter_column_chunking(sc, chunk, monkeypatch):
    """R split into L2-sized column chunks gives the same block (independent columns)."""
    monkeypatch.setenv("SC_CHUNK", chunk)
    g = scinputs.sbm(5000, 5, 12, 0.1, seed=21)
    L = laplacian.laplacian(g)
    lmax = 2.0 * float(g.degrees().max())
    X = scinputs.gaussian_block(1, g.n, 48)
    Y = gpu_filter(sc, g, X, 0.1 * lmax, lmax, 60, True)
    Yo = chebyshev.lowpass_filter(L, X.astype(np.float64), 0.1 * lmax, lmax, 60, True)
    assert rel(Y, Yo) <= F32_TOL


def test_filter_seeded_signals_and_host_buffers(sc):
    """X=NULL draws R on device from the seed (same numbers as scinputs); host in/out."""
    g = scinputs.sbm(2000, 5, 10, 0.1, seed=1234)
    G = sc.Graph.from_csr(g)
    lmax = 2.0 * float(g.degrees().max())
    Yh = np.zeros((g.n, 32), dtype=np.float32)
    sc.sc_filter_lowpass_f32(G.handle, 0.1 * lmax, lmax, 50, True, 32, 42, None, Yh)
    X = scinputs.gaussian_block(42, g.n, 32).astype(np.float64)
    Yo = chebyshev.lowpass_filter(laplacian.laplacian(g), X, 0.1 * lmax, lmax, 50, True)
    assert rel(Yh, Yo) <= F32_TOL


def test_filter_edgeless_and_constant_column(sc):
    # constant signal: F 1 = p(0) 1 (L 1 = 0) -- property valid at any size
    g = scinputs.sbm(20000, 10, 12, 0.1, seed=2)
    lmax = 2.0 * float(g.degrees().max())
    X = np.ones((g.n, 4), dtype=np.float32)
    Y = gpu_filter(sc, g, X, 0.05 * lmax, lmax, 80, True)
    p0 = np.polynomial.chebyshev.chebval(-1.0, chebyshev.filter_coeffs(0.05 * lmax, lmax, 80, True))
    assert np.allclose(Y, p0, rtol=2e-5, atol=2e-5)


def test_apply_general_coefficients(sc):
    g = scinputs.gmm_knn(3000, 6, 5, 8, seed=3)
    G = sc.Graph.from_csr(g)
    L = laplacian.laplacian(g)
    lmax = 2.0 * float(laplacian.strengths(laplacian.adjacency(g)).max())
    coeffs = np.random.default_rng(0).standard_normal(31) / np.arange(1, 32)
    X = scinputs.gaussian_block(5, g.n, 16)
    Xd = torch.from_numpy(X).cuda()
    Yd = torch.empty_like(Xd)
    sc.sc_filter_apply_f32(G.handle, coeffs, 30, lmax, 16, Xd, Yd)
    Yo = chebyshev.cheb_filter(L, X.astype(np.float64), coeffs, lmax)
    assert rel(Yd.cpu().numpy(), Yo) <= F32_TOL


def test_cheb_step_building_block_matches_filter(sc):
    """The per-step entry point used by the multi-GPU driver reproduces sc_filter_apply."""
    g = scinputs.sbm(3000, 4, 10, 0.1, seed=12)
    G = sc.Graph.from_csr(g)
    lmax = 2.0 * float(g.degrees().max())
    order, R = 25, 32
    d = chebyshev.filter_coeffs(0.1 * lmax, lmax, order, True)
    X = torch.from_numpy(scinputs.gaussian_block(8, g.n, R)).cuda()
    from paper_1509_08863_b200 import dist
    Y = dref.filter_local_steps(G.handle, d, order, lmax, X, row_split=(0, 1000, g.n))
    Yo = chebyshev.cheb_filter(laplacian.laplacian(g), X.cpu().numpy().astype(np.float64), d, lmax)
    assert rel(Y.cpu().numpy(), Yo) <= F32_TOL


@pytest.mark.slow
def test_full_size_c3_sampled_columns(sc):
    """BASELINE configs[3] at full size (N=1M, R=64, p=200) in the launch configuration
    bench.py times; the oracle recomputes two sampled columns (columns are independent)."""
    from scinputs import configs
    w = configs.WORKLOADS["c3_sbm1m"]
    g = configs.build_graph("c3_sbm1m")
    G = sc.Graph.from_csr(g)
    lmax = sc.sc_lambda_max(G.handle, 60, 0.01, 3)
    lc = 0.3 * lmax
    Yd = torch.empty((g.n, w.R), dtype=torch.float32, device="cuda")
    sc.sc_filter_lowpass_f32(G.handle, lc, lmax, w.order, w.jackson, w.R, 77, None, Yd)
    Y = Yd.cpu().numpy()
    X = scinputs.gaussian_block(77, g.n, w.R)
    cols = [0, 41]
    Yo = chebyshev.lowpass_filter(laplacian.laplacian(g), X[:, cols].astype(np.float64), lc, lmax, w.order, w.jackson)
    assert rel(Y[:, cols], Yo) <= F32_TOL


@pytest.mark.slow
def test_full_size_c1_all_columns(sc):
    """configs[1] (weighted Gaussian-mixture kNN, N=20k, R=24, p=100) at full size, every column."""
    from scinputs import configs
    w = configs.WORKLOADS["c1_gmm20k"]
    g = configs.build_graph("c1_gmm20k")
    G = sc.Graph.from_csr(g)
    L = laplacian.laplacian(g)
    lmax = lambda_max.lambda_max_bound(L, scinputs.gaussian_block(1, g.n, 1, dtype=np.float64)[:, 0], 300, 0.01)
    lc = 0.02 * lmax
    X = scinputs.gaussian_block(78, g.n, w.R)
    Y = gpu_filter(sc, g, X, lc, lmax, w.order, w.jackson, G=G)
    Yo = chebyshev.lowpass_filter(L, X.astype(np.float64), lc, lmax, w.order, w.jackson)
    assert rel(Y, Yo) <= F32_TOL


@pytest.mark.slow
@pytest.mark.parametrize("dtype,tol", [(torch.float32, F32_TOL), (torch.float64, F64_TOL)])
def test_full_size_c2_sampled_columns(sc, dtype, tol):
    """configs[2] (SBM N=100k, R=48, p=150) at full size in fp32 and fp64; three sampled columns."""
    from scinputs import configs
    w = configs.WORKLOADS["c2_sbm100k"]
    g = configs.build_graph("c2_sbm100k")
    G = sc.Graph.from_csr(g)
    lmax = sc.sc_lambda_max(G.handle, 60, 0.01, 3)
    lc = 0.05 * lmax
    X = scinputs.gaussian_block(79, g.n, w.R, dtype=np.float64)
    Y = gpu_filter(sc, g, X, lc, lmax, w.order, w.jackson, dtype=dtype, G=G)
    cols = [0, 17, 47]
    Xc = X[:, cols] if dtype == torch.float64 else X[:, cols].astype(np.float32).astype(np.float64)
    Yo = chebyshev.lowpass_filter(laplacian.laplacian(g), Xc, lc, lmax, w.order, w.jackson)
    assert rel(Y[:, cols], Yo) <= tol


@pytest.mark.slow
def test_full_size_c4_properties(sc):
    """configs[4] (SBM N=10M, ~2e8 nonzeros, R=96, p=300) at full size, in bench.py's launch
    configuration, checked by properties that hold at any size:
      * the constant vector is the lambda=0 eigenvector: F 1 = p(0) 1;
      * columns are independent: the filter of 8 sampled columns alone equals those columns of
        the full 96-column run (different chunking, same per-element arithmetic)."""
    from scinputs import configs
    w = configs.WORKLOADS["c4_sbm10m"]
    g = configs.build_graph("c4_sbm10m")
    G = sc.Graph.from_csr(g)
    n, R, p = g.n, w.R, w.order
    lmax = sc.sc_lambda_max(G.handle, 40, 0.01, 3)
    lc = 0.05 * lmax
    X = torch.empty((n, R), dtype=torch.float32, device="cuda")
    sc.sc_random_signals_f32(n, R, 0, 80, 0, 0.0, X)
    X[:, 5] = 1.0
    Y = torch.empty_like(X)
    sc.sc_filter_lowpass_f32(G.handle, lc, lmax, p, w.jackson, R, 0, X, Y)
    p0 = float(chebyshev.poly_eval(0.0, chebyshev.filter_coeffs(lc, lmax, p, w.jackson), lmax))
    c5 = Y[:, 5].double().cpu().numpy()
    assert np.max(np.abs(c5 - p0)) <= 1e-4 * max(1.0, abs(p0))
    cols = [0, 5, 31, 32, 63, 64, 90, 95]
    Xs = X[:, cols].contiguous()
    Ys = torch.empty_like(Xs)
    sc.sc_filter_lowpass_f32(G.handle, lc, lmax, p, w.jackson, len(cols), 0, Xs, Ys)
    torch.cuda.synchronize()
    a, b = Ys.cpu().numpy(), Y[:, cols].cpu().numpy()
    assert rel(a, b.astype(np.float64)) <= 1e-6


@pytest.mark.slow
def test_full_size_c4_oracle_columns(sc):
    """configs[4] (SBM N=10^7, 2e8 nonzeros, R=96, p=300) at full size in bench.py's launch
    configuration (96 columns, chunk plan 64 + 32): two sampled columns, one from each chunk,
    against the oracle's plain-C fp64 filter (oracle/cfilter.c, every host core)."""
    from oracle import cfilter
    from scinputs import configs
    w = configs.WORKLOADS["c4_sbm10m"]
    g = configs.build_graph("c4_sbm10m")
    G = sc.Graph.from_csr(g)
    n, R, p = g.n, w.R, w.order
    lmax = sc.sc_lambda_max(G.handle, 40, 0.01, 3)
    lc = 0.05 * lmax
    Y = torch.empty((n, R), dtype=torch.float32, device="cuda")
    sc.sc_filter_lowpass_f32(G.handle, lc, lmax, p, w.jackson, R, 81, None, Y)
    cols = [7, 90]
    Yg = Y[:, cols].cpu().numpy()
    del Y
    G.close()
    X = scinputs.gaussian_block(81, n, R, cols=cols).astype(np.float64)
    Yo = cfilter.cheb_filter(g, X, chebyshev.filter_coeffs(lc, lmax, p, w.jackson), lmax)
    assert rel(Yg, Yo) <= F32_TOL


def test_chunk_width_structural_choice(sc, monkeypatch):
    """filter_apply's chunk width on graphs of ~0.5-1M nodes (32-column chunks by the L2-budget
    rule): a power-law graph (max degree > 8x the mean) gets 64-column chunks -- the default run
    is bit-identical to SC_CHUNK=64 and SC_CHUNK_WIDE=0 to SC_CHUNK=32; the two widths agree to
    fp32 rounding (hub rows' chunk sums group edges by the width's lane groups, R15) and match
    the oracle on sampled columns."""
    g = scinputs.chung_lu(700_000, 20, 2.1, seed=11)
    G = sc.Graph.from_csr(g)
    R, order = 64, 30
    lmax = 2.0 * G.info()[3]
    d = chebyshev.filter_coeffs(0.05 * lmax, lmax, order, False)
    X = torch.from_numpy(scinputs.gaussian_block(8, g.n, R)).cuda()
    outs = {}
    for tag, env in (("32", {"SC_CHUNK": "32"}), ("64", {"SC_CHUNK": "64"}), ("auto", {}),
                     ("narrow", {"SC_CHUNK_WIDE": "0"})):
        for k in ("SC_CHUNK", "SC_CHUNK_WIDE"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        Y = torch.empty_like(X)
        sc.sc_filter_apply_f32(G.handle, d, order, lmax, R, X, Y)
        torch.cuda.synchronize()
        outs[tag] = Y.cpu().numpy()
    assert np.array_equal(outs["auto"], outs["64"])
    assert np.array_equal(outs["narrow"], outs["32"])
    assert rel(outs["32"], outs["64"]) <= 1e-6
    L = laplacian.laplacian(g)
    cols = [0, 37, 63]
    Yo = chebyshev.cheb_filter(L, X.cpu().numpy()[:, cols].astype(np.float64), d, lmax)
    for t in ("32", "64"):
        assert rel(outs[t][:, cols], Yo) <= F32_TOL


# ---------------------------------------------------------------------------
# eigencount moments and lambda_k dichotomy
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("sell", ["1", "0"])
def test_moments_counts_match_oracle(sc, sell, monkeypatch):
    """Eigencounts from the GPU moments (SELL kernel with exact fixed-point sums, or the CSR
    kernel's fixed-order partials) against the oracle's count on the same probes."""
    monkeypatch.setenv("SC_SELL", sell)
    g = scinputs.sbm(2000, 5, 10, 0.1, seed=1234)
    G = sc.Graph.from_csr(g)
    L = laplacian.laplacian(g)
    lmax = 1.01 * lambda_max.lambda_max_exact(L)
    order, npr = 50, 20
    P = scinputs.gaussian_block(4, g.n, npr, dtype=np.float64, stream=2)
    mu = sc.sc_cheb_moments(G.handle, lmax, order, npr, 0, torch.from_numpy(P).cuda())
    assert mu[0] == pytest.approx(np.sum(P * P), rel=1e-12)
    for ratio in [0.02, 0.07, 0.2, 0.5, 0.9]:
        c = sc.sc_eigencount_from_moments(mu, order, ratio * lmax, lmax, True)
        o = eigencount.count_below(L, ratio * lmax, lmax, order, P, True)
        assert abs(c - o) <= 1e-9 * mu[0]


@pytest.mark.parametrize("sell", ["1", "0"])
def test_moments_and_lambda_k_deterministic(sc, sell, monkeypatch):
    """Moments do not depend on the tile schedule -- SELL kernel: per-(warp, tile) partials
    summed as exact fixed-point integers (dynamic tiles); CSR kernel: static tile schedule,
    per-CTA partials summed in CTA order: repeated calls with the same seed give the same bits,
    at a size where many CTAs share the tiles; so does the lambda_k estimate built on them
    (ADVICE r01)."""
    monkeypatch.setenv("SC_SELL", sell)
    g = scinputs.sbm(150_000, 20, 16, 0.05, seed=8)
    G = sc.Graph.from_csr(g)
    lmax = 2.0 * G.info()[3]
    mus = [sc.sc_cheb_moments(G.handle, lmax, 60, 16, 42) for _ in range(3)]
    assert np.array_equal(mus[0], mus[1]) and np.array_equal(mus[0], mus[2])
    # the exact sums of the SELL path and the CSR path's rounded ones agree to fp64 rounding
    os.environ["SC_SELL"] = "0" if sell == "1" else "1"
    try:
        other = sc.sc_cheb_moments(G.handle, lmax, 60, 16, 42)
    finally:
        os.environ["SC_SELL"] = sell
    assert np.allclose(mus[0], other, rtol=0, atol=1e-11 * mus[0][0])
    lks = [sc.sc_estimate_lambda_k(G.handle, 20, lmax, 60, True, 16, 42, 40, 1e-4) for _ in range(2)]
    assert lks[0] == lks[1]


def test_lambda_k_dichotomy_matches_oracle(sc):
    g = scinputs.sbm(2000, 5, 10, 0.1, seed=1234)
    G = sc.Graph.from_csr(g)
    L = laplacian.laplacian(g)
    lmax = 1.01 * lambda_max.lambda_max_exact(L)
    order, npr = 50, 32
    P = scinputs.gaussian_block(9, g.n, npr, dtype=np.float64, stream=2)
    mu = sc.sc_cheb_moments(G.handle, lmax, order, npr, 0, torch.from_numpy(P).cuda())
    for k in [2, 5, 8]:
        lk, ck = sc.sc_lambda_k_from_moments(mu, order, k, lmax, True, 25, 1e-3)
        lo, co, trace = eigencount.estimate_lambda_k(L, k, lmax, order, P, True, 25, 1e-3)
        if lk != lo:   # only a decision within rounding of the threshold may differ
            assert min(abs(c - (k - 0.5)) for _, c in trace) < 1e-8 * mu[0]
        else:
            assert abs(ck - co) <= 1e-9 * mu[0]
    # seeded probes (stream 2) reproduce the host generator
    lk2, _ = sc.sc_estimate_lambda_k(G.handle, 5, lmax, order, True, npr, 9, 25, 1e-3)
    lo2, _, _ = eigencount.estimate_lambda_k(L, 5, lmax, order, P, True, 25, 1e-3)
    assert lk2 == lo2


# ---------------------------------------------------------------------------
# features, k-means, ARI
# ---------------------------------------------------------------------------

def test_normalize_rows(sc):
    F = scinputs.gaussian_block(3, 5000, 24)
    F[7] = 0.0
    Fd = torch.from_numpy(F.copy()).cuda()
    sc.sc_normalize_rows_f32(Fd, 5000, 24)
    ref = pipeline.normalize_rows(F).astype(np.float32)
    got = Fd.cpu().numpy()
    assert np.array_equal(got, ref) or np.max(np.abs(got - ref) / np.maximum(np.spacing(np.abs(ref)), 1e-45)) <= 1


def _features(seed, n, k, d, spread):
    rng = np.random.default_rng(seed)
    if spread < 0:   # integer grid: duplicate points, duplicate seeds, exactly tied distances
        return rng.integers(0, 3, (n, d)).astype(np.float32)
    C = rng.standard_normal((k, d))
    lab = rng.integers(0, k, n)
    return (C[lab] + spread * rng.standard_normal((n, d))).astype(np.float32)


@pytest.mark.parametrize("n,k,d,spread,restarts,max_iter", [
    (2000, 5, 32, 0.3, 10, 100), (20000, 10, 24, 0.8, 3, 100), (5000, 20, 48, 1.5, 2, 100), (3001, 7, 5, 0.5, 4, 100),
    # n*d >= 4e6 and n*k*d >= 2^27: concurrent restarts on worker streams + Hamerly pruning
    # (iterations capped so the fp64 oracle stays within ~a minute)
    pytest.param(90000, 32, 48, 1.0, 2, 12, marks=pytest.mark.slow),
    # same regime on integer-grid features: exact ties defeat the fp32 screen, so the
    # exact fp64 rescan of the ambiguous points decides them
    pytest.param(40000, 64, 56, -1.0, 1, 6, marks=pytest.mark.slow),
    # screened path with d and k off every tile multiple (29 dims, 70 centroids)
    pytest.param(70000, 70, 29, 0.7, 1, 6, marks=pytest.mark.slow),
    # tensor screen with rows wider than its register prefetch (d = 96: configs[4]'s width) and
    # with k = 200 (N = 208 columns of TMEM, 1 CTA per SM)
    pytest.param(30000, 40, 96, 0.8, 1, 6, marks=pytest.mark.slow),
    pytest.param(20000, 200, 96, 0.8, 1, 5, marks=pytest.mark.slow)])
def test_kmeans_bit_exact(sc, n, k, d, spread, restarts, max_iter):
    X = _features(n + k, n, k, d, spread)
    u = np.stack([scinputs.uniforms(7, k, offset=k * r) for r in range(restarts)])
    lab = torch.empty(n, dtype=torch.int32, device="cuda")
    C = np.zeros((k, d), dtype=np.float64)
    inertia, it, best = sc.sc_kmeans(torch.from_numpy(X).cuda(), n, d, k, restarts, max_iter, 0, u, lab, C)
    lo, Co, io, ito, ro, _ = kmeans.kmeans(X, k, u, max_iter)
    assert np.array_equal(lab.cpu().numpy(), lo)
    assert np.array_equal(C, Co)             # exactly rounded member sums -> identical centroids
    assert best == ro and it == ito
    assert inertia == pytest.approx(io, rel=1e-12)


@pytest.mark.parametrize("n,k,d,spread,restarts", [
    (90000, 32, 48, 0.8, 6),       # 16-byte staged rows
    (150000, 20, 29, -1.0, 4),     # d % 4 != 0 (4-byte staging), integer grid: ties, duplicate points
    (100000, 40, 64, 0.5, 17)])    # more restarts than one seeding batch (16)
def test_kmeans_batched_seeding_identical(sc, n, k, d, spread, restarts, monkeypatch):
    """Parallel restarts draw their k-means++ seeds in one batched pass (seed_batch: one launch
    per draw index for all restarts, rows read once): the result -- labels, centroids, inertia,
    iterations, best restart -- is bit-identical to every worker seeding its own restarts."""
    X = _features(n + 3 * k + d, n, k, d, spread)
    u = np.stack([scinputs.uniforms(11, k, offset=k * r) for r in range(restarts)])
    out = {}
    for batch in ("1", "0"):
        monkeypatch.setenv("SC_KMEANS_SEED_BATCH", batch)
        lab = torch.empty(n, dtype=torch.int32, device="cuda")
        C = np.zeros((k, d), dtype=np.float64)
        inertia, it, best = sc.sc_kmeans(torch.from_numpy(X).cuda(), n, d, k, restarts, 3, 0, u, lab, C)
        out[batch] = (lab.cpu().numpy(), C, inertia, it, best)
    a, b = out["1"], out["0"]
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert a[2] == b[2] and a[3] == b[3] and a[4] == b[4]


@pytest.mark.parametrize("n,k,d,spread", [
    (100, 2, 4, 0.5),        # one partial tile, N = 16 (k padded), K = 8 (d padded)
    (257, 17, 12, 0.4),      # tiles of 1-128 points, clusters of a few points
    (1000, 3, 8, -1.0),      # integer grid: ties everywhere -> the exact rescan decides
    (3000, 40, 64, 0.6),     # the register-prefetch staging at its widest (d = 64)
    (2000, 30, 68, 0.6),     # d = 68: 16-byte rows wider than the narrow prefetch
    (2500, 180, 100, 0.6),   # k x d that allow one CTA per SM: the wide (32-chunk) prefetch, two tiles per CTA
    (1500, 9, 20, 0.05)])    # tight clusters: most points decided, few change
def test_kmeans_screens_forced_small(sc, n, k, d, spread, monkeypatch):
    """The screens (tensor-core and fp32) and the Hamerly check forced on small problems
    (thresholds 0): edge shapes of the tiles / panels / queues, labels, centroids, iteration
    count and best restart identical to the fp64 oracle (R8)."""
    monkeypatch.setenv("SC_KMEANS_SCREEN_MIN", "0")
    monkeypatch.setenv("SC_KMEANS_PRUNE_MIN", "0")
    X = _features(n + 7 * k + d, n, k, d, spread)
    restarts, max_iter = 3, 30
    u = np.stack([scinputs.uniforms(3, k, offset=k * r) for r in range(restarts)])
    lo, Co, io, ito, ro, _ = kmeans.kmeans(X, k, u, max_iter)
    for tc, wide, pair in (("1", "1", "1"), ("1", "1", "0"), ("1", "0", "1"), ("0", "1", "1")):
        monkeypatch.setenv("SC_KMEANS_TC", tc)
        monkeypatch.setenv("SC_KMEANS_TC_WIDE", wide)
        monkeypatch.setenv("SC_KMEANS_TC_PAIR", pair)
        lab = torch.empty(n, dtype=torch.int32, device="cuda")
        C = np.zeros((k, d), dtype=np.float64)
        inertia, it, best = sc.sc_kmeans(torch.from_numpy(X).cuda(), n, d, k, restarts, max_iter, 0, u, lab, C)
        assert np.array_equal(lab.cpu().numpy(), lo), tc
        assert np.array_equal(C, Co) and best == ro and it == ito, tc
        assert inertia == pytest.approx(io, rel=1e-12)


def test_kmeans_unaligned_features_same_labels(sc):
    """Features whose base pointer is not 16-byte aligned (a view one float into its storage)
    take the 4-byte staging path of the per-point kernels; d % 4 == 0 aligned features the
    16-byte path: both give the oracle's labels."""
    n, k, d = 40000, 110, 32      # n*k*d >= 2^27: fp32 screen and Hamerly check on
    X = _features(n + 3, n, k, d, 0.9)
    u = np.stack([scinputs.uniforms(13, k, offset=k * r) for r in range(2)])
    lo, Co, io, ito, ro, _ = kmeans.kmeans(X, k, u, 8)
    big = torch.zeros(n * d + 1, dtype=torch.float32, device="cuda")
    big[1:] = torch.from_numpy(X).cuda().reshape(-1)
    for F in (torch.from_numpy(X).cuda(), big[1:].view(n, d)):
        assert (F.data_ptr() % 16 == 0) == (F.storage_offset() == 0)
        lab = torch.empty(n, dtype=torch.int32, device="cuda")
        C = np.zeros((k, d), dtype=np.float64)
        inertia, it, best = sc.sc_kmeans(F, n, d, k, 2, 8, 0, u, lab, C)
        assert np.array_equal(lab.cpu().numpy(), lo)
        assert np.array_equal(C, Co) and best == ro and it == ito


@pytest.mark.parametrize("case", ["k1", "k_eq_n", "d1", "three_distinct_rows"])
def test_kmeans_edge_cases(sc, case):
    """Degenerate k-means inputs: one cluster, one point per cluster, one dimension, and
    fewer distinct points than clusters (D^2 total reaches 0 -> uniform draws, duplicate
    centres, empty clusters keep their centre, tied distances -> lowest index)."""
    rng = np.random.default_rng(11)
    if case == "k1":
        X, k = rng.standard_normal((50, 3)).astype(np.float32), 1
    elif case == "k_eq_n":
        X, k = rng.standard_normal((40, 2)).astype(np.float32), 40
    elif case == "d1":
        X, k = rng.standard_normal((300, 1)).astype(np.float32), 5
    else:
        base = rng.standard_normal((3, 4)).astype(np.float32)
        X, k = base[rng.integers(0, 3, 200)], 5
    n, d = X.shape
    u = np.stack([scinputs.uniforms(5, k, offset=k * r) for r in range(3)])
    lab = torch.empty(n, dtype=torch.int32, device="cuda")
    C = np.zeros((k, d), dtype=np.float64)
    inertia, it, best = sc.sc_kmeans(torch.from_numpy(X).cuda(), n, d, k, 3, 100, 0, u, lab, C)
    lo, Co, io, ito, ro, _ = kmeans.kmeans(X, k, u, 100)
    assert np.array_equal(lab.cpu().numpy(), lo)
    assert np.array_equal(C, Co)
    assert best == ro and it == ito
    assert inertia == pytest.approx(io, rel=1e-12, abs=1e-300)


def test_kmeans_on_filtered_features_and_default_uniforms(sc):
    """Shared deterministic seeding: uniforms from the counter generator (NULL)."""
    g = scinputs.sbm(2000, 5, 10, 0.1, seed=1234)
    L = laplacian.laplacian(g)
    lmax = 1.01 * lambda_max.lambda_max_exact(L)
    X = scinputs.gaussian_block(3, g.n, 32).astype(np.float64)
    F = chebyshev.lowpass_filter(L, X, 0.08 * lmax, lmax, 50, True).astype(np.float32)
    lab = np.zeros(g.n, dtype=np.int32)
    inertia, it, best = sc.sc_kmeans(F, g.n, 32, 5, 10, 100, 123, None, lab)
    u = np.stack([scinputs.uniforms(123, 5, offset=5 * r) for r in range(10)])
    lo, _, io, _, ro, _ = kmeans.kmeans(F, 5, u, 100)
    assert np.array_equal(lab, lo) and best == ro


def test_kmeans_full_size_properties(sc):
    """configs[3]-sized k-means (10^6 x 64, k = 100: fp32 screen, Hamerly checks, incremental
    exact updates, concurrent restarts) checked by properties the oracle can compute at this
    size: sampled labels are the exact fp64 argmin (oracle arithmetic, lowest index on ties)
    under the returned centroids, sampled centroids are the correctly rounded member means,
    and the inertia is the oracle's sum of exact distances."""
    import math
    rng = np.random.default_rng(77)
    n, d, k = 1_000_000, 64, 100
    centers = rng.standard_normal((k, d)) * 0.5
    X = (centers[rng.integers(0, k, n)] + rng.standard_normal((n, d))).astype(np.float32)
    lab = torch.empty(n, dtype=torch.int32, device="cuda")
    C = np.zeros((k, d), dtype=np.float64)
    u = np.stack([scinputs.uniforms(3, k, offset=k * r) for r in range(2)])
    inertia, it, best = sc.sc_kmeans(torch.from_numpy(X).cuda(), n, d, k, 2, 8, 0, u, lab, C)
    L = lab.cpu().numpy()
    idx = rng.choice(n, 3000, replace=False)
    D = kmeans.sq_dists(X[idx], C)
    assert np.array_equal(L[idx], np.argmin(D, axis=1))
    # centroids of the final assignment: the member means of the labels the last update used
    # differ from L only if the run stopped at max_iter; check the converged-or-not invariant
    # through the exact dmin instead, plus member means when converged
    Xd = X.astype(np.float64)
    dm = np.zeros(n)
    for q in range(d):
        diff = Xd[:, q] - C[L, q]
        dm += diff * diff
    assert inertia == pytest.approx(math.fsum(dm), rel=1e-12)
    if it < 8:   # converged: C are the exact member means of L
        for c in rng.choice(k, 4, replace=False):
            M = Xd[L == c]
            if len(M):
                want = np.array([math.fsum(M[:, q]) / len(M) for q in range(d)])
                assert np.array_equal(C[c], want)


def test_ari_matches_oracle(sc):
    rng = np.random.default_rng(0)
    for n, ka, kb in [(1000, 5, 7), (100000, 20, 20), (10, 1, 1), (4, 2, 2)]:
        a = rng.integers(0, ka, n).astype(np.int32)
        b = rng.integers(0, kb, n).astype(np.int32)
        assert sc.sc_ari(a, b, n) == pytest.approx(oari.ari(a, b), abs=1e-12)
    assert sc.sc_ari(np.array([0, 0, 1, 1], np.int32), np.array([0, 1, 0, 1], np.int32), 4) == pytest.approx(-0.5)


# ---------------------------------------------------------------------------
# pipeline
# ---------------------------------------------------------------------------

def test_cluster_pipeline_recovers_planted_sbm(sc):
    # configs[0]'s own graph (avg degree 10, eps 0.1) is NOT recoverable by spectral
    # clustering on the combinatorial Laplacian: its lambda_2..lambda_5 interleave with
    # modes localised on low-degree nodes, and exact classical SC scores ARI 0.0 there
    # (reading R11).  A denser SBM of the same size is recovered exactly.
    g = scinputs.sbm(2000, 5, 20, 0.05, seed=1234)
    G = sc.Graph.from_csr(g)
    lab = np.zeros(g.n, dtype=np.int32)
    info = sc.sc_cluster(G.handle, 5, 32, 60, True, 32, 2024, 10, 100, False, lab)
    assert oari.ari(lab, g.labels) > 0.95
    assert 4.5 <= info[2] <= 5.5
    ev = np.linalg.eigvalsh(laplacian.laplacian_dense(g))
    assert ev[-1] <= info[0] <= 1.02 * ev[-1]


@pytest.mark.parametrize("normalize", [False, True])
def test_cluster_matches_oracle_pipeline(sc, normalize):
    """sc_cluster (§4.1 steps 1-6, l.303-329) against oracle.pipeline.accelerated_sc
    fed the same inputs: the GPU's lambda_max bound (two estimators of one bound, R3), the
    eigencount probes (stream 2, seed ^ 0x5e5e5e5e, variance 1/n_probe), the signal block
    (stream 0, fp32-rounded), the k-means++ uniforms (stream 1).  Checked stage by stage:
    lambda~_k equal (or the dichotomy decision within rounding of k - 1/2), the features at
    the fp32 tolerance, k-means labels bit-exact on the oracle's fp32-rounded features, and
    the end-to-end labels (ARI >= 0.99)."""
    g = scinputs.sbm(2000, 5, 20, 0.05, seed=1234)
    k, R, order, npr, seed, restarts, max_iter = 5, 32, 60, 32, 2024, 10, 100
    G = sc.Graph.from_csr(g)
    lab = np.zeros(g.n, dtype=np.int32)
    info = sc.sc_cluster(G.handle, k, R, order, True, npr, seed, restarts, max_iter, normalize, lab)
    lmax, lk = float(info[0]), float(info[1])
    X = scinputs.gaussian_block(seed, g.n, R).astype(np.float64)
    P = scinputs.gaussian_block(seed ^ 0x5E5E5E5E, g.n, npr, dtype=np.float64, stream=2)
    u = np.stack([scinputs.uniforms(seed, k, offset=k * r) for r in range(restarts)])
    out = pipeline.accelerated_sc(g, k, X, P, order, True, u, lambda_max_value=lmax, normalize=normalize,
                                  max_iter=max_iter, bisect_iter=40, bisect_rtol=1e-4)
    L = laplacian.laplacian(g)
    if lk != out["lambda_k"]:
        _, _, trace = eigencount.estimate_lambda_k(L, k, lmax, order, P, True, 40, 1e-4)
        assert min(abs(c - (k - 0.5)) for _, c in trace) < 1e-8 * np.sum(P * P)
    # features: the filter call sc_cluster makes (seeded signals, lambda~_k, Jackson)
    Yd = torch.empty((g.n, R), dtype=torch.float32, device="cuda")
    sc.sc_filter_lowpass_f32(G.handle, lk, lmax, order, True, R, seed, None, Yd)
    Yo = chebyshev.lowpass_filter(L, X, lk, lmax, order, True)
    assert rel(Yd.cpu().numpy(), Yo) <= F32_TOL
    # k-means on the oracle's features, rounded to fp32 once: labels bit-exact
    F = (pipeline.normalize_rows(Yo) if normalize else Yo).astype(np.float32)
    lab2 = np.zeros(g.n, dtype=np.int32)
    _, it2, best2 = sc.sc_kmeans(F, g.n, R, k, restarts, max_iter, seed, None, lab2)
    lo, _, _, ito, ro, _ = kmeans.kmeans(F, k, u, max_iter)
    assert np.array_equal(lab2, lo) and best2 == ro and it2 == ito
    # end to end
    assert oari.ari(lab, out["labels"]) >= 0.99
    assert oari.ari(lab, g.labels) > 0.95


# ---------------------------------------------------------------------------
# filter order m* (§2.4 Eq. (4) l.151-162, §4.1 step 3 l.312; reading R18)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("ratio,jackson,delta,theta,n_grid", [
    (1.0, False, 0.1, 0.1, 10000), (1.0, True, 0.1, 0.1, 10000), (0.5, False, 0.1, 0.1, 10000),
    (0.5, True, 0.1, 0.1, 10000), (0.1, False, 0.1, 0.1, 10000), (0.1, True, 0.1, 0.1, 10000),
    (0.03, False, 0.1, 0.1, 10000), (0.02, False, 0.05, 0.2, 3001), (0.3, True, 0.02, 0.05, 5000),
    (0.77, False, 0.1, 0.1, 10000), (0.01, False, 0.1, 0.1, 10000), (0.2, True, 0.1, 0.0, 2)])
def test_filter_order_matches_oracle(sc, ratio, jackson, delta, theta, n_grid):
    """sc_filter_order (device Clenshaw over the grid, orders in batches) against
    oracle.chebyshev.minimal_order (trigonometric form, one order at a time): the same m*, and
    the grid error of m* equal to fp64 rounding.  Cases span batch boundaries (m* 1 .. ~150), a
    tighter delta, a wider / no band, and a 2-point grid."""
    m, err = sc.sc_filter_order(ratio, delta, jackson, theta, n_grid, 400)
    mo = chebyshev.minimal_order(ratio, delta, jackson, 400, theta, n_grid)
    assert m == (mo or 0)
    if mo:
        assert err == pytest.approx(chebyshev.approx_error(ratio, mo, jackson, theta, n_grid), abs=1e-10)
        if mo > 1:    # not within rounding of delta, so the integer decision is unambiguous
            assert chebyshev.approx_error(ratio, mo - 1, jackson, theta, n_grid) > delta + 1e-9


def test_filter_order_none_found(sc):
    """No order meets delta: m* = 0 and the error of the last order tried (theta = 0 with the cut on
    the grid: the jump is between neighbouring grid points, reading R18)."""
    m, err = sc.sc_filter_order(0.5, 0.1, False, 0.0, 10001, 100)
    assert m == 0 and chebyshev.minimal_order(0.5, 0.1, False, 100, 0.0, 10001) is None
    assert err == pytest.approx(chebyshev.approx_error(0.5, 100, False, 0.0, 10001), abs=1e-10)


@pytest.mark.parametrize("jackson", [False, True])
def test_cluster_with_selected_order_matches_oracle(sc, jackson):
    """sc_cluster with order < 0 (§4.1 step 3, l.312): lambda~_k estimated at |order|,
    then the filter at m*(lambda~_k/lambda_N; 0.1); the order it reports equals the oracle's m*
    at the same lambda ratio, and the labels agree with the oracle pipeline run the same way."""
    g = scinputs.sbm(2000, 5, 20, 0.05, seed=1234)
    k, R, npr, seed, restarts, max_iter = 5, 32, 32, 2024, 10, 100
    G = sc.Graph.from_csr(g)
    lab = np.zeros(g.n, dtype=np.int32)
    info = sc.sc_cluster(G.handle, k, R, -60, jackson, npr, seed, restarts, max_iter, False, lab)
    lmax, lk, used = float(info[0]), float(info[1]), int(info[6])
    want = chebyshev.minimal_order(min(1.0, lk / lmax), 0.1, jackson, 2000) or 2000
    assert used == want
    X = scinputs.gaussian_block(seed, g.n, R).astype(np.float64)
    P = scinputs.gaussian_block(seed ^ 0x5E5E5E5E, g.n, npr, dtype=np.float64, stream=2)
    u = np.stack([scinputs.uniforms(seed, k, offset=k * r) for r in range(restarts)])
    out = pipeline.accelerated_sc(g, k, X, P, -60, jackson, u, lambda_max_value=lmax, max_iter=max_iter,
                                  bisect_iter=40, bisect_rtol=1e-4)
    if out["lambda_k"] == lk:
        assert out["order"] == used
    assert oari.ari(lab, out["labels"]) >= 0.99
    # the same order given explicitly reproduces the labels bit for bit
    lab2 = np.zeros(g.n, dtype=np.int32)
    info2 = sc.sc_cluster(G.handle, k, R, used, jackson, npr, seed, restarts, max_iter, False, lab2)
    if info2[1] == lk:
        assert np.array_equal(lab, lab2)


# ---------------------------------------------------------------------------
# stability measure gamma(k) (§4.3 Eq.(11))
# ---------------------------------------------------------------------------

def _oracle_stability(g, ks, lks, lmax, J, R, order, jackson, seed, restarts, max_iter):
    from oracle import stability
    L = laplacian.laplacian(g)
    out, labs = {}, {}
    for k, lk in zip(ks, lks):
        ls = []
        for j in range(J):
            X = scinputs.gaussian_block(seed + j, g.n, R).astype(np.float64)
            F = chebyshev.lowpass_filter(L, X, lk, lmax, order, jackson).astype(np.float32)
            u = np.stack([scinputs.uniforms(seed + j, k, offset=k * r) for r in range(restarts)])
            ls.append(kmeans.kmeans(F, k, u, max_iter)[0])
        out[k] = stability.gamma(ls)
        labs[k] = ls
    return out, labs


def test_stability_matches_oracle(sc):
    g = scinputs.sbm(1200, 4, 20, 0.03, seed=21)
    L = laplacian.laplacian(g)
    lmax = lambda_max.lambda_max_exact(L) * 1.01
    ev = np.linalg.eigvalsh(L.toarray())
    ks = [2, 3, 4, 5, 6]
    lks = [0.5 * (ev[k - 1] + ev[k]) for k in ks]          # mid-gap cuts from the dense oracle
    J, R, order, seed, restarts, max_iter = 4, 12, 60, 77, 3, 100
    G = sc.Graph.from_csr(g)
    lab = np.zeros((len(ks), J, g.n), dtype=np.int32)
    gam, lk_used = sc.sc_stability(G.handle, ks[0], ks[-1], J, R, order, True, 0, seed, restarts, max_iter,
                                   lambda_max=lmax, lambda_k=np.array(lks), labels=lab)
    assert np.array_equal(lk_used, lks)
    want, wlabs = _oracle_stability(g, ks, lks, lmax, J, R, order, True, seed, restarts, max_iter)
    for c, k in enumerate(ks):
        agree = [oari.ari(lab[c, j], wlabs[k][j]) for j in range(J)]
        assert min(agree) > 0.99, (k, agree)
        assert gam[c] == pytest.approx(want[k], abs=2e-3)
    # the planted k = 4 is the global maximum (§4.3 l.361-362)
    assert ks[int(np.argmax(gam))] == 4 and gam[ks.index(4)] > 0.99


def test_stability_estimated_cuts_and_j2(sc):
    g = scinputs.sbm(1500, 3, 20, 0.02, seed=5)
    G = sc.Graph.from_csr(g)
    gam, lk = sc.sc_stability(G.handle, 2, 4, 2, 8, 60, True, 24, 9, 2, 100)
    assert np.all(np.diff(lk) >= 0) and np.all(lk > 0)
    lab = np.zeros((3, 2, g.n), dtype=np.int32)
    gam2, _ = sc.sc_stability(G.handle, 2, 4, 2, 8, 60, True, 24, 9, 2, 100, labels=lab)
    assert np.array_equal(gam, gam2)                          # deterministic
    for c in range(3):                                        # J = 2: gamma is one ARI
        assert gam[c] == pytest.approx(oari.ari(lab[c, 0], lab[c, 1]), abs=1e-12)
    assert int(np.argmax(gam)) + 2 == 3


def test_stability_screened_workers_match_exact_scan(sc, monkeypatch):
    """At a size where the k-means screens run (n k d >= 3e7: tensor screen, fp32 screen, exact
    scan of their ambiguous points) with concurrent workers of different k: labels and gamma
    identical to the plain exact scan with one worker (R8 bit-exactness; regression for a
    shared-memory attribute lowered by one worker under another's launch)."""
    g = scinputs.sbm(80_000, 10, 16, 0.05, seed=31)
    G = sc.Graph.from_csr(g)
    args = (G.handle, 9, 12, 2, 48, 60, True, 24, 5, 2, 30)
    lab = np.zeros((4, 2, g.n), dtype=np.int32)
    gam, lk = sc.sc_stability(*args, labels=lab)
    monkeypatch.setenv("SC_KMEANS_SCREEN", "0")
    monkeypatch.setenv("SC_KMEANS_PRUNE_MIN", "1e30")
    monkeypatch.setenv("SC_STABILITY_WORKERS", "1")
    lab2 = np.zeros((4, 2, g.n), dtype=np.int32)
    gam2, lk2 = sc.sc_stability(*args, labels=lab2)
    assert np.array_equal(lk, lk2)
    assert np.array_equal(lab, lab2)
    assert np.array_equal(gam, gam2)


def test_row_partitioned_steps_emulated_two_ranks(sc):
    """The multi-GPU data path on one GPU without inter-rank waiting: both ranks' local CSR
    (renumbered columns, interior-first rows, halo block), per-step halo fill from the
    owner's send list, interior then boundary fused steps -- vs the oracle on the whole graph."""
    from paper_1509_08863_b200 import dist as pdist
    g = scinputs.sbm(2400, 4, 10, 0.05, seed=31)
    world, R, order = 2, 16, 30
    parts = [pdist.local_part(g.row_ptr, g.col_idx, g.values, g.n, r, world) for r in range(world)]
    halos = [p.halo_gid for p in parts]
    for p in parts:
        pdist.send_lists_from_halos(p, halos)
    Gs = [sc.Graph(p.n_local, p.row_ptr, p.col_idx, p.values, n_cols=p.n_local + p.n_halo) for p in parts]
    fns = [dref.cuda_step_fn(G.handle) for G in Gs]
    lmax = 2.0 * float(g.degrees().max())
    d = chebyshev.filter_coeffs(0.12 * lmax, lmax, order, True)
    X = scinputs.gaussian_block(41, g.n, R)
    T0, bufs, Ys, sends = [], [], [], []
    for p in parts:
        t = torch.zeros((p.n_local + p.n_halo, R), dtype=torch.float32, device="cuda")
        t[: p.n_local] = torch.from_numpy(X[p.r0:p.r1]).cuda()[torch.from_numpy(p.perm).cuda()]
        T0.append(t)
        bufs.append([torch.zeros_like(t) for _ in range(2)])
        Ys.append(torch.empty((p.n_local, R), dtype=torch.float32, device="cuda"))
        off = np.concatenate([[0], np.cumsum(p.send_counts)])
        sends.append({q: torch.from_numpy(p.send_idx[off[q]:off[q + 1]]).cuda() for q in range(world)})
    for st in dref.step_schedule(order, d, lmax):
        s = st["s"]
        cur = [T0[r] if s == 0 else bufs[r][s & 1] for r in range(world)]
        prev = [None if s == 0 else (T0[r] if s == 1 else bufs[r][(s - 1) & 1]) for r in range(world)]
        nxt = [bufs[r][(s + 1) & 1] if st["store_next"] else None for r in range(world)]
        for r, p in enumerate(parts):            # halo exchange (emulated: device copies)
            blocks = [cur[q][sends[q][r]] for q in range(world) if q != r]
            if p.n_halo:
                cur[r][p.n_local:] = torch.cat(blocks)
        for r, p in enumerate(parts):
            fns[r](0, p.n_interior, prev[r], cur[r], nxt[r], Ys[r], st)
            fns[r](p.n_interior, p.n_local, prev[r], cur[r], nxt[r], Ys[r], st)
    torch.cuda.synchronize()
    Yfull = np.zeros((g.n, R))
    for r, p in enumerate(parts):
        y = np.empty((p.n_local, R))
        y[p.perm] = Ys[r].cpu().numpy()
        Yfull[p.r0:p.r1] = y
    Yo = chebyshev.cheb_filter(laplacian.laplacian(g), X.astype(np.float64), d, lmax)
    assert all(p.n_halo > 0 and 0 < p.n_interior < p.n_local for p in parts)
    assert rel(Yfull, Yo) <= F32_TOL


def _dist_group(sc, g, world):
    """All `world` ranks' partition plans held by this process (sc_comm_local: the library's
    single-process emulation -- halo rows copied between the ranks' buffers, sums in rank
    order)."""
    from paper_1509_08863_b200 import dist as pdist
    parts = [pdist.local_part(g.row_ptr, g.col_idx, g.values, g.n, r, world) for r in range(world)]
    halos = [p.halo_gid for p in parts]
    for p in parts:
        pdist.send_lists_from_halos(p, halos)
    Gs = [sc.Graph(p.n_local, p.row_ptr, p.col_idx, p.values, n_cols=p.n_local + p.n_halo) for p in parts]
    comms = [sc.sc_comm_local(world, r) for r in range(world)]
    plans = [sc.sc_dist_create(G.handle, c, p.n_interior, p.send_idx, np.asarray(p.send_counts, np.int64),
                               np.asarray(p.recv_counts, np.int64)) for G, c, p in zip(Gs, comms, parts)]
    return parts, Gs, comms, plans


@pytest.mark.parametrize("world", [1, 2, 3])
def test_partitioned_lambda_estimates_emulated(sc, world):
    """PAPER.md §4.1 steps 1-2 on a row-partitioned graph (sc_dist_lambda_max,
    sc_dist_cheb_moments, sc_dist_estimate_lambda_k): lambda^_N is a tight upper bound of the
    exact lambda_N; the eigencounts of the moments and the dichotomy's lambda~_k match the
    oracle on the probes the ranks drew (assembled in global row order)."""
    g = scinputs.sbm(2000, 5, 10, 0.1, seed=1234)
    parts, Gs, comms, plans = _dist_group(sc, g, world)
    try:
        if world > 1:
            assert all(p.n_halo > 0 for p in parts)
        row0 = [p.r0 for p in parts]
        L = laplacian.laplacian(g)
        lN = lambda_max.lambda_max_exact(L)
        lm = sc.sc_dist_lambda_max(plans, 60, 0.01, 7, row0)
        assert lN <= lm <= 1.02 * lN
        lmax, order, npr, seed = 1.01 * lN, 50, 20, 4
        mu = sc.sc_dist_cheb_moments(plans, lmax, order, npr, seed, row0)
        P = np.zeros((g.n, npr))
        for p in parts:
            P[p.r0 + p.perm] = scinputs.gaussian_block(seed, p.n_local, npr, row0=p.r0, dtype=np.float64, stream=2)
        assert mu[0] == pytest.approx(np.sum(P * P), rel=1e-12)
        for ratio in [0.02, 0.07, 0.2, 0.5, 0.9]:
            c = sc.sc_eigencount_from_moments(mu, order, ratio * lmax, lmax, True)
            o = eigencount.count_below(L, ratio * lmax, lmax, order, P, True)
            assert abs(c - o) <= 1e-9 * mu[0]
        for k in [2, 5, 8]:
            lk, ck = sc.sc_dist_estimate_lambda_k(plans, k, lmax, order, True, npr, seed, row0, 25, 1e-3)
            lo, co, trace = eigencount.estimate_lambda_k(L, k, lmax, order, P, True, 25, 1e-3)
            if lk != lo:
                assert min(abs(c - (k - 0.5)) for _, c in trace) < 1e-8 * mu[0]
            else:
                assert abs(ck - co) <= 1e-9 * mu[0]
    finally:
        for pl in plans:
            sc.sc_dist_free(pl)
        for c in comms:
            sc.sc_comm_free(c)


@pytest.mark.parametrize("world,n,k,d,restarts,spread,force", [
    (1, 2000, 4, 6, 2, 0.5, False), (2, 3000, 5, 8, 3, 0.5, False), (3, 20000, 12, 16, 2, 1.0, False),
    (4, 40000, 32, 48, 2, 1.0, False),
    # screens (tensor-core, fp32 for the first assignment) and the Hamerly check forced on
    # every rank's rows
    (3, 20000, 12, 16, 2, 1.0, True), (4, 40000, 32, 48, 2, 1.0, True)])
def test_dist_kmeans_emulated_bit_exact(sc, world, n, k, d, restarts, spread, force, monkeypatch):
    """sc_dist_kmeans (§4.1 step 6 on a row partition): all ranks held by this
    process (sc_comm_local; one host thread and stream per rank, reductions at a host
    rendezvous), uneven row blocks, against the oracle on the rank-major concatenation:
    labels, centroids, iteration count and best restart bit-exact (exact integer member sums
    reduced over the ranks; `force`: the screened and pruned assignment paths)."""
    if force:
        monkeypatch.setenv("SC_KMEANS_SCREEN_MIN", "0")
        monkeypatch.setenv("SC_KMEANS_PRUNE_MIN", "0")
    rng = np.random.default_rng(n + k)
    centers = rng.standard_normal((k, d)) * 2.0
    X = (centers[rng.integers(0, k, n)] + spread * rng.standard_normal((n, d))).astype(np.float32)
    cuts = np.sort(rng.choice(np.arange(1, n), world - 1, replace=False)) if world > 1 else np.array([], int)
    bounds = np.concatenate([[0], cuts, [n]]).astype(int)
    comms = [sc.sc_comm_local(world, r) for r in range(world)]
    try:
        Fs = [torch.from_numpy(np.ascontiguousarray(X[bounds[r]:bounds[r + 1]])).cuda() for r in range(world)]
        labs = [torch.full((bounds[r + 1] - bounds[r],), -1, dtype=torch.int32, device="cuda") for r in range(world)]
        u = np.stack([scinputs.uniforms(9, k, offset=k * r) for r in range(restarts)])
        C = np.zeros((k, d))
        inertia, it, best = sc.sc_dist_kmeans(comms, Fs, d, k, restarts, 100, 0, u, labs, C)
        lab = np.concatenate([x.cpu().numpy() for x in labs])
        lo, Co, io, ito, ro, _ = kmeans.kmeans(X, k, u, 100)
        assert np.array_equal(lab, lo)
        assert np.array_equal(C, Co)
        assert best == ro and it == ito
        assert inertia == pytest.approx(io, rel=1e-12)
    finally:
        for c in comms:
            sc.sc_comm_free(c)


@pytest.mark.parametrize("world,normalize", [(2, False), (3, True)])
def test_partitioned_pipeline_emulated(sc, world, normalize):
    """PAPER.md §4.1 steps 1-6 on a row partition held by this process (dist.P2PGroup.cluster:
    sc_dist_lambda_max, sc_dist_estimate_lambda_k, the fused-exchange filter, row
    normalisation, sc_dist_kmeans) against the single-GPU sc_cluster on the same graph and
    seed: lambda estimates agree to estimator accuracy, the partitions agree (ARI >= 0.99) and
    recover the planted communities."""
    from paper_1509_08863_b200 import dist as pdist
    g = scinputs.sbm(3000, 5, 20, 0.05, seed=17)
    k, R, order, npr, seed, restarts = 5, 32, 60, 32, 77, 5
    G = sc.Graph.from_csr(g)
    lab1 = np.zeros(g.n, dtype=np.int32)
    info1 = sc.sc_cluster(G.handle, k, R, order, True, npr, seed, restarts, 100, normalize, lab1)
    grp = pdist.P2PGroup(g.row_ptr, g.col_idx, g.values, g.n, world, R)
    try:
        labs, info = grp.cluster(k, R, order, True, npr, seed, restarts, 100, normalize)
        torch.cuda.synchronize()
        lab = np.zeros(g.n, dtype=np.int32)
        for p, l in zip(grp.parts, labs):
            lab[p.r0 + p.perm] = l.cpu().numpy()
    finally:
        grp.close()
    ev = np.linalg.eigvalsh(laplacian.laplacian_dense(g))
    assert ev[-1] <= info["lambda_max"] <= 1.02 * ev[-1]
    assert info["lambda_max"] == pytest.approx(info1[0], rel=1e-3)
    assert 4.5 <= info["count_k"] <= 5.5
    assert oari.ari(lab, lab1) >= 0.99
    assert oari.ari(lab, g.labels) > 0.95


@pytest.mark.parametrize("sell", ["1", "0"])
@pytest.mark.parametrize("world,R,chunk,waits", [(2, 16, None, False), (3, 6, None, False), (4, 16, "8", False),
                                                 (2, 12, "4", False), (1, 8, None, False), (3, 16, "8", True)])
def test_p2p_fused_exchange_emulated(sc, world, R, chunk, waits, sell, monkeypatch):
    """The fused-exchange filter (sc_p2p_*): every rank's step kernel stores its boundary rows
    of T_{s+1} straight into the peers' halos.  All ranks held by this process on one GPU
    (sc_p2p_filter_group_f32: dependency-ordered launches on one stream, nothing waits), incl.
    several column chunks, a ragged R and world 1 -- vs the oracle on the whole graph.  Both
    step kernels carry the exchange epilogue: the SELL kernel (default) and the CSR kernel."""
    from paper_1509_08863_b200 import dist as pdist
    monkeypatch.setenv("SC_SELL", sell)
    if chunk:
        monkeypatch.setenv("SC_CHUNK", chunk)
    if waits:   # also run the flag waits of the multi-process path (each already satisfied)
        monkeypatch.setenv("SC_P2P_GROUP_WAITS", "1")
    g = scinputs.sbm(3000, 6, 10, 0.1, seed=21)
    order = 30
    L = laplacian.laplacian(g)
    lmax = 2.0 * float(g.degrees().max())
    d = chebyshev.filter_coeffs(0.15 * lmax, lmax, order, True)
    X = scinputs.gaussian_block(4, g.n, R)
    grp = pdist.P2PGroup(g.row_ptr, g.col_idx, g.values, g.n, world, R)
    try:
        Xs = [torch.from_numpy(np.ascontiguousarray(X[p.r0:p.r1][p.perm])).cuda() for p in grp.parts]
        Ys = [torch.full_like(x, float("nan")) for x in Xs]
        for _ in range(2):                     # twice: call-spanning signal counters, buffer reuse
            grp.filter(d, order, lmax, Xs, Ys)
            torch.cuda.synchronize()
            Y = np.zeros((g.n, R))
            for p, y in zip(grp.parts, Ys):
                Y[p.r0 + p.perm] = y.cpu().numpy()
            Yo = chebyshev.cheb_filter(L, X.astype(np.float64), d, lmax)
            assert rel(Y, Yo) <= F32_TOL
        if world > 1:
            assert all(p.n_halo > 0 for p in grp.parts)
    finally:
        grp.close()


@pytest.mark.parametrize("world,hub", [(2, "8"), (3, "4"), (2, "100000")])
def test_p2p_fused_exchange_weighted_split_rows(sc, world, hub, monkeypatch):
    """The SELL kernel's fused-exchange epilogue on a weighted graph with hub rows: rows above
    the split threshold (SC_SELL_HUB_DEG) are summed in chunks by hub_chunk_kernel and still
    stored into the peers' halos by the epilogue; two column chunks (SC_CHUNK 8, R = 16)."""
    from paper_1509_08863_b200 import dist as pdist
    monkeypatch.setenv("SC_SELL_HUB_DEG", hub)
    monkeypatch.setenv("SC_CHUNK", "8")
    base = scinputs.random_connected(1500, 0.01, seed=9, weighted=True)
    # a star on top: node 0 joined to every 3rd node (degree ~500: a split row)
    src = np.repeat(np.arange(base.n), np.diff(base.row_ptr))
    keep = src < base.col_idx
    star = np.arange(3, base.n, 3)
    g = scinputs.from_edges(base.n, np.concatenate([src[keep], np.zeros(star.size, np.int64)]),
                            np.concatenate([base.col_idx[keep], star]),
                            np.concatenate([base.values[keep], np.full(star.size, 0.7, np.float32)]))
    assert g.degrees()[0] > 400
    R, order = 16, 25
    L = laplacian.laplacian(g)
    lmax = 2.0 * float(L.diagonal().max())   # Gershgorin: 2 max_i s_i
    d = chebyshev.filter_coeffs(0.1 * lmax, lmax, order, False)
    X = scinputs.gaussian_block(6, g.n, R)
    grp = pdist.P2PGroup(g.row_ptr, g.col_idx, g.values, g.n, world, R)
    try:
        Xs = [torch.from_numpy(np.ascontiguousarray(X[p.r0:p.r1][p.perm])).cuda() for p in grp.parts]
        Ys = [torch.full_like(x, float("nan")) for x in Xs]
        grp.filter(d, order, lmax, Xs, Ys)
        torch.cuda.synchronize()
        Y = np.zeros((g.n, R))
        for p, y in zip(grp.parts, Ys):
            Y[p.r0 + p.perm] = y.cpu().numpy()
        assert rel(Y, chebyshev.cheb_filter(L, X.astype(np.float64), d, lmax)) <= F32_TOL
    finally:
        grp.close()


@pytest.mark.parametrize("world,n_cg,R", [(4, 2, 16), (8, 2, 24), (2, 2, 8)])
def test_column_x_row_grid_emulated(sc, world, n_cg, R):
    """The 2-D decomposition bench.py uses on N GPUs (dist.grid_shape): column group c filters
    columns column_range(R, n_cg, c) of every row; its world/n_cg ranks row-partition the graph
    with the fused peer-store exchange among themselves only.  Each column group's ranks are
    emulated on this GPU (sc_p2p_filter_group_f32); the assembled block vs the oracle."""
    from paper_1509_08863_b200 import dist as pdist
    g = scinputs.sbm(2400, 6, 10, 0.1, seed=22)
    order = 25
    lmax = 2.0 * float(g.degrees().max())
    d = chebyshev.filter_coeffs(0.15 * lmax, lmax, order, True)
    X = scinputs.gaussian_block(6, g.n, R)
    cg, n_row = pdist.grid_shape(world, R, min_cols=4, col_groups=n_cg)
    Y = np.full((g.n, R), np.nan)
    for c in range(cg):
        c0, c1 = pdist.column_range(R, cg, c)
        grp = pdist.P2PGroup(g.row_ptr, g.col_idx, g.values, g.n, n_row, c1 - c0)
        try:
            Xs = [torch.from_numpy(np.ascontiguousarray(X[p.r0:p.r1, c0:c1][p.perm])).cuda() for p in grp.parts]
            Ys = [torch.full_like(x, float("nan")) for x in Xs]
            grp.filter(d, order, lmax, Xs, Ys)
            torch.cuda.synchronize()
            for p, y in zip(grp.parts, Ys):
                Y[p.r0 + p.perm, c0:c1] = y.cpu().numpy()
        finally:
            grp.close()
    Yo = chebyshev.cheb_filter(laplacian.laplacian(g), X.astype(np.float64), d, lmax)
    assert not np.isnan(Y).any()
    assert rel(Y, Yo) <= F32_TOL


def test_p2p_filter_single_rank_host_buffers(sc):
    """sc_p2p_filter_f32 (the multi-process entry point: chunk-start waits, T_0 push,
    signalled steps) on a 1-rank partition with host X / Y, incl. a ragged R."""
    from paper_1509_08863_b200 import dist as pdist
    g = scinputs.sbm(2500, 3, 12, 0.05, seed=34)
    part = pdist.local_part(g.row_ptr, g.col_idx, g.values, g.n, 0, 1)
    part = pdist.send_lists_from_halos(part, [part.halo_gid])
    G = sc.Graph(part.n_local, part.row_ptr, part.col_idx, part.values, n_cols=part.n_local + part.n_halo)
    pf = pdist.P2PFilter(part, G.handle, g.n, 32)
    lmax = 2.0 * float(g.degrees().max())
    L = laplacian.laplacian(g)
    try:
        for R, order in [(32, 25), (13, 7)]:
            d = chebyshev.filter_coeffs(0.1 * lmax, lmax, order, True)
            X = scinputs.gaussian_block(6, g.n, R)
            Xp = np.ascontiguousarray(X[part.perm])
            Yp = np.zeros_like(Xp)
            pf.filter(d, order, lmax, Xp, Yp)
            Y = np.empty((g.n, R))
            Y[part.perm] = Yp
            Yo = chebyshev.cheb_filter(L, X.astype(np.float64), d, lmax)
            assert rel(Y, Yo) <= F32_TOL
    finally:
        pf.close()


def _ipc_worker(rank, world, port, q):
    import torch.distributed as tdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch as th
        th.cuda.set_device(0)
        import paper_1509_08863_b200 as scm
        from paper_1509_08863_b200 import dist as pdist
        g = scinputs.sbm(1200, 3, 8, 0.1, seed=8)
        part = pdist.exchange_send_lists(pdist.local_part(g.row_ptr, g.col_idx, g.values, g.n, rank, world))
        G = scm.Graph(part.n_local, part.row_ptr, part.col_idx, part.values, n_cols=part.n_local + part.n_halo)
        pf = pdist.P2PFilter(part, G.handle, g.n, 8)     # export, all-gather, cudaIpcOpenMemHandle
        tdist.barrier()
        pf.close()
        tdist.barrier()
        q.put((rank, True))
    except Exception as e:
        q.put((rank, repr(e)))
    finally:
        tdist.destroy_process_group()


def test_p2p_ipc_handles_map_across_processes(sc):
    """Two processes exchange and open each other's CUDA IPC handles (the mapping step of
    the multi-GPU path; both on this GPU, so no filter runs: its steps would wait on each
    other)."""
    import socket
    import torch.multiprocessing as tmp
    s_ = socket.socket()
    s_.bind(("127.0.0.1", 0))
    port = s_.getsockname()[1]
    s_.close()
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(240)
        assert p.exitcode == 0
    res = dict(q.get(timeout=10) for _ in range(2))
    assert res == {0: True, 1: True}, res


def test_nccl_dist_filter_single_rank(sc):
    """sc_dist_filter_f32 end to end on one rank (NCCL communicator of size 1, no halo):
    the library-side multi-GPU schedule against the oracle, incl. a ragged R."""
    from paper_1509_08863_b200 import dist as pdist
    g = scinputs.sbm(3000, 3, 12, 0.05, seed=33)
    part = pdist.local_part(g.row_ptr, g.col_idx, g.values, g.n, 0, 1)
    pdist.send_lists_from_halos(part, [part.halo_gid])
    G = sc.Graph(part.n_local, part.row_ptr, part.col_idx, part.values, n_cols=part.n_local + part.n_halo)
    nf = pdist.NcclFilter(part, G.handle)
    lmax = 2.0 * float(g.degrees().max())
    L = laplacian.laplacian(g)
    for R, order in [(32, 25), (13, 7)]:
        d = chebyshev.filter_coeffs(0.1 * lmax, lmax, order, True)
        X = scinputs.gaussian_block(5, g.n, R)
        Xp = torch.from_numpy(X[part.perm]).cuda()
        Yp = torch.empty_like(Xp)
        nf.filter(d, order, lmax, Xp, Yp)
        torch.cuda.synchronize()
        Y = np.empty((g.n, R))
        Y[part.perm] = Yp.cpu().numpy()
        Yo = chebyshev.cheb_filter(L, X.astype(np.float64), d, lmax)
        assert rel(Y, Yo) <= F32_TOL
    nf.close()


# ---------------------------------------------------------------------------
# randomised filter cases: sizes, degrees, weights, widths, orders, both kernels
# ---------------------------------------------------------------------------

def _random_case(i):
    rng = np.random.default_rng(1000 + i)
    n = int(rng.integers(2, 6000))
    if rng.random() < 0.5:
        g = scinputs.random_connected(min(n, 1500), float(rng.uniform(0.0, 0.02)), seed=int(rng.integers(1 << 30)),
                                      weighted=bool(rng.random() < 0.5))
    else:
        k = int(rng.integers(1, 8))
        n = max(n, 4 * k + 4)
        g = scinputs.sbm(n, k, float(rng.uniform(2.0, 25.0)), float(rng.uniform(0.0, 0.3)),
                         seed=int(rng.integers(1 << 30)))
    R = int(rng.choice([1, 2, 3, 4, 5, 7, 8, 12, 13, 16, 24, 31, 32, 48, 64, 96, 100, 128, 130]))
    order = int(rng.integers(1, 60))
    return g, R, order, bool(rng.random() < 0.5), float(rng.uniform(0.01, 1.0))


@pytest.mark.parametrize("path", list(PATHS))
@pytest.mark.parametrize("i", range(16))
def test_filter_random_cases(sc, i, path, monkeypatch):
    _path_env(monkeypatch, path)
    g, R, order, jackson, ratio = _random_case(i)
    L = laplacian.laplacian(g)
    lmax = 2.0 * float(max(laplacian.strengths(laplacian.adjacency(g)).max(), 1e-12))
    X = scinputs.gaussian_block(50 + i, g.n, R)
    Y = gpu_filter(sc, g, X, ratio * lmax, lmax, order, jackson)
    Yo = chebyshev.lowpass_filter(L, X.astype(np.float64), ratio * lmax, lmax, order, jackson)
    assert rel(Y, Yo) <= F32_TOL, (g.n, g.nnz, R, order)


# ---------------------------------------------------------------------------
# bench.py contract on the GPU (small workload): the single-GPU line and the partitioned path
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("extra", [[], ["--dist-path"], ["--dist-path", "--exchange", "nccl"]])
def test_bench_json_line_gpu(sc, extra):
    """`bench.py` prints one JSON line with the driver's keys, a positive roofline from the
    per-launch events (also on the partitioned paths, whose SELL steps record them) and a
    positive kernel count -- on configs[2] (100k nodes: streaming kernels, L2 flushed)."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--workload", "c2_sbm100k", "--steps", "3",
                        "--warmup", "3", "--no-cluster", "--no-stability", "--no-cpu-baseline", *extra],
                       capture_output=True, text=True, timeout=900, cwd=root,
                       env=dict(os.environ, MASTER_ADDR="127.0.0.1", SC_RESIDENT="0"))
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "roofline", "clocks", "e2e",
                "gpu_launches", "config"):
        assert key in d, key
    assert d["value"] > 0 and d["gpu_launches"] > 0
    assert d["roofline"]["achieved"] > 0 and 0 < d["roofline"]["frac"] < 1.5


def test_bench_exchange_selftest_child(sc):
    """`bench.py`'s multi-GPU arm first runs the fused peer-store exchange against the NCCL
    exchange in a child process (`--selftest-exchange`, spawned by `p2p_selftest_child` with its
    own MASTER_PORT and without torchrun's agent-store variables) and falls back to NCCL if the
    child fails.  On the one GPU here: the child as the parent spawns it, with one rank -- it
    must rendezvous on the shifted port, run both exchanges and exit 0."""
    import importlib.util
    import types
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(root, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    env = dict(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1", MASTER_PORT="29611",
               TORCHELASTIC_USE_AGENT_STORE="True")
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        ok, why = bench.p2p_selftest_child(types.SimpleNamespace(gpus=1, seed=1234), timeout_s=600)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    assert ok, why
