/*
 * sc_b200.h -- C ABI of the B200-native accelerated spectral clustering hot path.
 *
 * Paper: N. Tremblay, G. Puy, P. Borgnat, R. Gribonval, P. Vandergheynst,
 * "Accelerated spectral clustering using graph filtering of random signals"
 * (arXiv:1509.08863), cited below as PAPER.md §x / line y.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - Return value: SC_OK (0) on success, a negative SC_ERR_* code otherwise;
 *    sc_last_error() returns a human-readable message for the calling thread.
 *    On error no output is guaranteed to be written.
 *  - Pointers: every array argument may live in host memory (pageable or pinned)
 *    or in CUDA device memory of the current device; the library detects which
 *    with cudaPointerGetAttributes and copies host arrays in/out itself (so the
 *    same call serves an end-to-end host-buffer caller and a device-resident
 *    caller).  The caller keeps ownership of every array it passes.
 *  - Dense blocks (signals, filtered output, features) are row-major
 *    n x R arrays (row i = node i, column q = signal q), contiguous.
 *  - Graphs are symmetric CSR of the weighted adjacency W (§2 lines
 *    59-63): row_ptr int64[n+1], col_idx int32[nnz] (no diagonal entries),
 *    values float32[nnz] or NULL for a unit-weight ("pattern") graph.
 *  - stream: a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Calls that return host scalars synchronise that stream before returning.
 *  - Precision: "_f32" paths store and accumulate in fp32, "_f64" paths in fp64.
 *    k-means decisions (argmin, D^2 sampling, best replicate) are taken in fp64.
 *  - There is no CPU fallback: without a CUDA device every compute call
 *    returns SC_ERR_CUDA.
 *  - A graph handle owns grow-only device workspaces and per-shape launch plans:
 *    use one handle from one host thread / one stream at a time (distinct handles
 *    are independent).
 */
#ifndef SC_B200_H
#define SC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SC_OK            0
#define SC_ERR_ARG      -1   /* invalid argument (sizes, ranges, null pointers)   */
#define SC_ERR_CUDA     -2   /* CUDA runtime error or no device                    */
#define SC_ERR_STATE    -3   /* handle in the wrong state                          */
#define SC_ERR_NOMEM    -4   /* device or host allocation failed                   */

typedef struct sc_graph sc_graph;   /* opaque device-resident graph + workspace */

/* Version of the ABI (major*10000 + minor*100 + patch). */
int sc_version(void);

/* Message describing the last error raised on the calling thread ("" if none). */
const char* sc_last_error(void);

/* ------------------------------------------------------------------------ */
/* Graph                                                                    */
/* ------------------------------------------------------------------------ */

/*
 * sc_graph_load -- upload W and build the combinatorial Laplacian operator
 * L = S - W, S = diag(s), s_i = sum_{j != i} W_ij (§2.1 lines 66-72).
 *
 *  n_rows   rows of W held by this process (all N nodes on one GPU; the local
 *           row block of a row-partitioned multi-GPU run).
 *  n_cols   number of distinct column indices the rows reference
 *           (= N on one GPU; local rows + halo rows when partitioned; col_idx < n_cols).
 *  nnz      stored entries = row_ptr[n_rows].
 *  row_ptr, col_idx, values   CSR arrays as above (values may be NULL: unit weights).
 *  out      receives the new handle; free it with sc_graph_free.
 * The strengths s_i are computed on device in fp64 from the rows as given.
 * Errors: SC_ERR_ARG for n_rows<1, n_cols<n_rows, nnz<0, null arrays, row_ptr[0] != 0,
 *         row_ptr[n_rows] != nnz, decreasing row_ptr, column index outside [0, n_cols);
 *         SC_ERR_NOMEM / SC_ERR_CUDA on device failures.
 */
int sc_graph_load(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* row_ptr,
                  const int32_t* col_idx, const float* values, sc_graph** out);

int sc_graph_free(sc_graph* g);

/* n_rows, n_cols, nnz and max_i s_i (Gershgorin: lambda_N <= 2 max s_i). */
int sc_graph_info(const sc_graph* g, int64_t* n_rows, int64_t* n_cols, int64_t* nnz,
                  double* max_strength);

/* Copy the fp64 strengths s (n_rows values) to `out` (host or device). */
int sc_graph_strengths(const sc_graph* g, double* out, void* stream);

/* ------------------------------------------------------------------------ */
/* Spectral bounds and filter design (§2.4, §4.1 steps 1 and 3)    */
/* ------------------------------------------------------------------------ */

/*
 * sc_lambda_max -- upper bound of lambda_N, the largest eigenvalue of L
 * (§4.1 step 1, line 309: "Estimate L's largest eigenvalue").
 * Runs `iters` Lanczos steps (fp64, start vector from the counter-based
 * generator with `seed`), takes the largest Ritz value theta and returns
 * min((1+margin)*theta, 2*max_i s_i)  (the Chebyshev domain must contain the
 * whole spectrum; 2 max s_i is Gershgorin's bound).  Single-GPU graphs only
 * (n_cols == n_rows).  Errors: SC_ERR_ARG for iters<1 or margin<0.
 */
int sc_lambda_max(sc_graph* g, int iters, double margin, uint64_t seed, double* out,
                  void* stream);

/*
 * sc_cheby_coeffs -- host: the order+1 coefficients d_j = g_j c_j of the
 * Chebyshev approximation of the ideal low-pass h_{lambda_c}(lambda) =
 * 1[lambda <= lambda_c] on [0, lambda_max] (Eq. (2) line 128 and
 * §2.4):  c_0 = 1 - theta/pi,  c_j = -2 sin(j theta)/(pi j),
 * theta = arccos(2 lambda_c/lambda_max - 1);  g_j = Jackson damping factors
 * when `jackson` != 0 (else 1).  coeffs: host array of order+1 doubles.
 * Errors: SC_ERR_ARG for order<0, lambda_max<=0.
 */
int sc_cheby_coeffs(double lambda_c, double lambda_max, int order, int jackson, double* coeffs);

/*
 * sc_filter_order -- m*(lambda_c/lambda_N; delta), the filter order of PAPER.md §2.4
 * "Note on the choice of m" (Eq. (4)) used by §4.1 step 3 (line 312): the
 * smallest m in [1, m_max] whose polynomial (the coefficients sc_cheby_coeffs gives for
 * lambda_c = ratio, lambda_max = 1, `jackson`) satisfies |h_ratio(l) - p_m(l)| <= delta at
 * every point l of the grid {i/(n_grid-1)} U {i min(1, 2 ratio)/(n_grid-1)}, i < n_grid,
 * outside the transition band [ratio(1-theta), ratio(1+theta)] (reading R18: the
 * sup over the whole interval is >= 1/2 for any polynomial at the jump).  The paper fixes
 * delta = 0.1 (line 162); R18 takes theta = 0.1, n_grid = 10000.
 * Evaluated on the device (fp64 Clenshaw, orders tried in batches of increasing size on
 * `stream`; the call synchronises the stream).
 *  m_star  host int: m*, or 0 if no order <= m_max meets delta.
 *  err     host double or NULL: the grid error of m* (of the last order tried when m* = 0).
 * Errors: SC_ERR_ARG for ratio outside (0, 1], delta <= 0, theta outside [0, 1),
 *         n_grid outside [2, 2^24], m_max outside [1, 4096]; SC_ERR_CUDA.
 */
int sc_filter_order(double ratio, double delta, int jackson, double theta, int n_grid, int m_max,
                    int* m_star, double* err, void* stream);

/* ------------------------------------------------------------------------ */
/* Random signals (§3.1, §4.1 step 4 line 316)       */
/* ------------------------------------------------------------------------ */

/*
 * sc_random_signals -- rows [row0, row0+n) of the N x R block of i.i.d.
 * N(0, variance) entries of the counter-based generator (splitmix64 +
 * Box-Muller in fp64); variance <= 0 means
 * 1/R (the paper's 1/eta).  stream_id: 0 = signals, 2 = eigencount probes.
 * out: n x R, fp32 (_f32) or fp64 (_f64), host or device.
 */
int sc_random_signals_f32(int64_t n, int R, int64_t row0, uint64_t seed, int stream_id,
                          double variance, float* out, void* stream);
int sc_random_signals_f64(int64_t n, int R, int64_t row0, uint64_t seed, int stream_id,
                          double variance, double* out, void* stream);

/* ------------------------------------------------------------------------ */
/* The hot path: fused Chebyshev filter (§2.4 Eq. (3), §4.1 step 5) */
/* ------------------------------------------------------------------------ */

/*
 * sc_filter_apply -- Y = sum_{j=0}^{order} coeffs[j] T_j(L~) X, L~ = (2/lambda_max) L - I,
 * by the three-term recurrence T_{j+1} = 2 L~ T_j - T_{j-1}, each step one fused
 * CSR SpMM that also accumulates Y (O(m(|E|+N))).
 *  X   n x R input block (signals), Y  n x R output block; X and Y must not alias.
 *  coeffs  host array of order+1 doubles (e.g. from sc_cheby_coeffs).
 *  order >= 1, R >= 1, lambda_max > 0.  Single-GPU graphs only (n_cols == n_rows).
 */
int sc_filter_apply_f32(sc_graph* g, const double* coeffs, int order, double lambda_max,
                        int R, const float* X, float* Y, void* stream);
int sc_filter_apply_f64(sc_graph* g, const double* coeffs, int order, double lambda_max,
                        int R, const double* X, double* Y, void* stream);

/*
 * sc_filter_lowpass -- the paper's fast filtering of random signals
 * (§4.1 steps 3-5, Eq. (10)): coefficients of h_{lambda_c} (with
 * optional Jackson damping) applied to X.  If X is NULL the N x R signal block
 * is drawn on device from `seed` (sc_random_signals, variance 1/R) first.
 * Y receives the n x R filtered block F R whose rows are the features f~_i.
 */
int sc_filter_lowpass_f32(sc_graph* g, double lambda_c, double lambda_max, int order,
                          int jackson, int R, uint64_t seed, const float* X, float* Y,
                          void* stream);
int sc_filter_lowpass_f64(sc_graph* g, double lambda_c, double lambda_max, int order,
                          int jackson, int R, uint64_t seed, const double* X, double* Y,
                          void* stream);

/*
 * sc_cheb_step -- one fused recurrence step on caller-owned device buffers, for
 * the row-partitioned multi-GPU driver (rows [row_begin, row_end) of this
 * rank's block; gathers read T_cur rows 0..n_cols-1, i.e. local + halo rows):
 *    T_next = a * (L T_cur) + b_cur * T_cur + b_prev * T_prev
 *    Y      (y_mode 1: =, 2: +=)  cy_prev T_prev + cy_cur T_cur + cy_next T_next
 * T_prev may be NULL when b_prev == 0 and cy_prev == 0; T_next may be NULL to
 * skip storing it (last step).  ld_* are row strides in elements.  All
 * pointers device, fp32.
 */
int sc_cheb_step_f32(sc_graph* g, int64_t row_begin, int64_t row_end, int R,
                     const float* T_prev, int64_t ld_prev, const float* T_cur, int64_t ld_cur,
                     float* T_next, int64_t ld_next, float* Y, int64_t ld_y,
                     double a, double b_cur, double b_prev, double cy_prev, double cy_cur,
                     double cy_next, int y_mode, void* stream);

/* ------------------------------------------------------------------------ */
/* lambda_k estimation (§3.2)                        */
/* ------------------------------------------------------------------------ */

/*
 * sc_cheb_moments -- mu_m = <X, T_m(L~) X>_F for m = 0..2*order from `order`
 * recurrence steps (T_{2j} = 2 T_j^2 - I, T_{2j+1} = 2 T_j T_{j+1} - T_1), fp64.
 * X: n x R probes (host/device, fp64) or NULL = drawn from `seed` (stream 2,
 * variance 1/R).  moments: 2*order+1 doubles (host or device).
 */
int sc_cheb_moments(sc_graph* g, double lambda_max, int order, int R, uint64_t seed,
                    const double* X, double* moments, void* stream);

/*
 * sc_eigencount -- estimated number of eigenvalues <= lambda_c:
 * ||F_{lambda_c} X||_F^2 evaluated from the moments (host arithmetic).
 */
int sc_eigencount_from_moments(const double* moments, int order, double lambda_c,
                               double lambda_max, int jackson, double* count);

/*
 * sc_estimate_lambda_k -- dichotomy on [0, lambda_max] keeping
 * count(lo) < k - 1/2 <= count(hi) (reading R6) until
 * hi - lo <= rtol*lambda_max or max_iter; returns lambda_k = hi and count(hi).
 * All counts come from ONE moments pass (n_probe probe columns, seed).
 */
int sc_estimate_lambda_k(sc_graph* g, int k, double lambda_max, int order, int jackson,
                         int n_probe, uint64_t seed, int max_iter, double rtol,
                         double* lambda_k, double* count_k, void* stream);

/* Same dichotomy on precomputed moments (host only; k-scans reuse one pass). */
int sc_lambda_k_from_moments(const double* moments, int order, int k, double lambda_max,
                             int jackson, int max_iter, double rtol, double* lambda_k,
                             double* count_k);

/* ------------------------------------------------------------------------ */
/* Features and k-means (§2.2 step 4, §4.1 step 6)                 */
/* ------------------------------------------------------------------------ */

/* f_i <- f_i / ||f_i||_2 in place (rows of zero norm stay zero); fp32. */
int sc_normalize_rows_f32(float* F, int64_t n, int d, void* stream);

/*
 * sc_kmeans -- best of `restarts` k-means runs on the n x d fp32 features F.
 * Replicate r seeds with k-means++ using uniforms u[r*k + t] (t < k): taken
 * from `uniforms` (host/device, restarts*k doubles) or, if NULL, from the
 * counter-based generator (seed, stream 1, counters r*k + t).  Lloyd: assign
 * argmin_c sum_q (x_q - C_cq)^2 in fp64 (ascending q, no FMA contraction,
 * lowest c on ties), update to member means (empty cluster keeps its centre),
 * stop when an assignment repeats or after max_iter updates.  Lowest inertia
 * wins, ties -> lowest r.
 *  labels    n int32 (host/device);   centroids  k*d doubles or NULL;
 *  inertia   host double or NULL;     iters      host int or NULL;
 *  best_restart host int or NULL.
 * Errors: SC_ERR_ARG for k<1, k>n, d<1, d>200 (the assignment kernel stages 64 points and
 * 64 centroids of d fp64 coordinates in shared memory), restarts<1, max_iter<1, n >= 2^25.
 */
int sc_kmeans(const float* F, int64_t n, int d, int k, int restarts, int max_iter,
              uint64_t seed, const double* uniforms, int32_t* labels, double* centroids,
              double* inertia, int* iters, int* best_restart, void* stream);

/* Adjusted Rand index of two labelings of n nodes (§4.3, §5). */
int sc_ari(const int32_t* a, const int32_t* b, int64_t n, double* out, void* stream);

/* ------------------------------------------------------------------------ */
/* Whole pipeline (§4.1 steps 1-6)                                 */
/* ------------------------------------------------------------------------ */

/*
 * sc_cluster -- lambda_max (Lanczos), lambda_k (moments + dichotomy, n_probe
 * probes, Jackson), filter R random signals at lambda_k (order, jackson),
 * optional row normalisation, k-means (restarts).  labels: n int32.
 * order > 0: steps 2 and 5 use this order.  order < 0: step 2 uses -order and step 5
 * the order m*(lambda~_k/lambda_N; 0.1) of sc_filter_order (theta 0.1, 10000-point grid,
 * 2000 if no order <= 2000 meets delta) -- PAPER.md §4.1 step 3, line 312.
 * info (host, may be NULL): 7 doubles [lambda_max, lambda_k, count_k, inertia,
 * kmeans_iters, best_restart, filter order used].
 * The eigencount of step 2 always uses the Jackson-damped polynomial, whatever
 * `jackson` says: the count ||F X||^2 estimates #{lambda_l <= lambda_c} only if
 * the polynomial stays in [0, 1] (R5); the undamped truncated series
 * overshoots (Gibbs) and would bias the count.  `jackson` selects the filter of
 * step 5 only.  Random draws: Lanczos start (seed ^ 0x1a2b3c4d), probes (stream 2,
 * seed ^ 0x5e5e5e5e), signals (stream 0, seed), k-means++ uniforms (stream 1, seed).
 */
int sc_cluster(sc_graph* g, int k, int R, int order, int jackson, int n_probe,
               uint64_t seed, int restarts, int max_iter, int normalize, int32_t* labels,
               double* info, void* stream);

/*
 * sc_stability -- stability measure for the number of clusters (§4.3,
 * Eq.(11)): for every k in [k_min, k_max], J clusterings from J
 * independent draws of the R random signals (replicate j draws R with seed + j,
 * stream 0, variance 1/R) and
 *     gamma(k) = 2/(J(J-1)) * sum_{a<b} ari(C^a_k, C^b_k)          (R7).
 * Each replicate runs the Chebyshev recurrence once (order fused steps, all
 * order+1 terms T_m kept in device memory: (order+1)*n*ceil4(R)*4 bytes) and
 * forms the filtered block of every cut lambda_k from it, then k-means with k
 * clusters (`restarts` k-means++ replicates, uniforms from seed + j, stream 1).
 *  lambda_max  > 0: the Chebyshev domain; <= 0: Lanczos estimate (as sc_lambda_max, 60 steps, 1%).
 *  lambda_k    host array of K = k_max-k_min+1 cuts, or NULL: estimated from one moments
 *              pass of n_probe probes (seed ^ 0x5e5e5e5e, stream 2), Jackson-damped
 *              counts, dichotomy as sc_lambda_k_from_moments (40 steps, rtol 1e-4).
 *  gamma       host double[K] (out);  lambda_k_out host double[K] or NULL (out: cuts used).
 *  labels      NULL or int32 [K][J][n] (host or device; out): every clustering.
 * Single-GPU graphs only.  Errors: SC_ERR_ARG for 1 <= k_min <= k_max < n, J >= 2,
 * R >= 1, order >= 1, restarts >= 1, max_iter >= 1 violated; SC_ERR_NOMEM when the
 * T_m stack does not fit.
 */
int sc_stability(sc_graph* g, int k_min, int k_max, int J, int R, int order, int jackson, int n_probe,
                 uint64_t seed, int restarts, int max_iter, double lambda_max, const double* lambda_k,
                 double* gamma, double* lambda_k_out, int32_t* labels, void* stream);

/* ------------------------------------------------------------------------ */
/* Row-partitioned multi-GPU filter (north_star: halo exchange over NVLink   */
/* with NCCL, overlapped with the interior SpMM)                             */
/* ------------------------------------------------------------------------ */

typedef struct sc_comm sc_comm;   /* NCCL communicator + communication stream */
typedef struct sc_dist sc_dist;   /* one rank's partition plan                */

/* 128-byte NCCL unique id (rank 0 creates it; the caller broadcasts it). */
int sc_nccl_unique_id(void* id);

/* Communicator of `world` ranks on the current device.  Errors: SC_ERR_CUDA from NCCL. */
int sc_comm_init(const void* id, int world, int rank, sc_comm** out);
/* Communicator without NCCL for rank `rank` of `world` (<= 8): the single-process emulation
 * in which one process holds every rank's plan on one GPU (sc_dist_lambda_max and friends
 * with nheld == world).  Errors: SC_ERR_ARG for world outside [1, 8] or a bad rank. */
int sc_comm_local(int world, int rank, sc_comm** out);
int sc_comm_free(sc_comm* c);

/*
 * sc_dist_create -- partition plan of this rank.  g is the rank's local CSR loaded with
 * sc_graph_load(n_local, n_local + n_halo, ...): rows in local order with the
 * n_interior rows that have no remote neighbour first; columns [0, n_local) local rows,
 * [n_local, n_local + n_halo) halo rows grouped by owner rank (ascending).
 * send_idx (host/device int64, n_send): local row positions to send, grouped by peer;
 * send_counts / recv_counts (host int64, world): rows sent to / received from each rank
 * (sum(recv_counts) must equal n_halo).  dist.py builds all of these.
 */
int sc_dist_create(sc_graph* g, sc_comm* c, int64_t n_interior, const int64_t* send_idx, int64_t n_send,
                   const int64_t* send_counts, const int64_t* recv_counts, sc_dist** out);
int sc_dist_free(sc_dist* d);

/*
 * sc_dist_filter_f32 -- this rank's rows of Y = sum_j coeffs[j] T_j(L~) X (as
 * sc_filter_apply_f32), X and Y the n_local x R blocks in the plan's local row order.
 * Each recurrence step: pack the send rows, exchange halos with NCCL send/recv on the
 * communicator's stream, run the interior rows' fused step concurrently, then the
 * boundary rows.  All ranks must call it with the same coeffs/order/lambda_max/R.
 */
int sc_dist_filter_f32(sc_dist* d, const double* coeffs, int order, double lambda_max, int R, const float* X,
                       float* Y, void* stream);

/*
 * Row-partitioned lambda estimates (§4.1 steps 1-2, l.309-311; §3.2 l.269-275):
 * the single-GPU estimators (sc_lambda_max, sc_cheb_moments, sc_estimate_lambda_k) on the
 * partition, every SpMV preceded by the halo exchange of its vector and every inner product
 * summed over the ranks.  ds / nheld: the plans this process holds -- nheld = 1 (one process
 * per GPU; a multi-rank plan needs an NCCL communicator: halos by send/recv, sums by
 * ncclAllReduce) or nheld = world (all ranks of the partition in this process on one GPU,
 * created with sc_comm_local: halos copied, sums in rank order; ds[r] is rank r).
 * row0 (host int64 [nheld] or NULL = 0): counter offset of each held rank's first local row
 * for the start vector (stream 0) and the probes (stream 2, variance 1/n_probe, counters
 * (row0 + i) * n_probe + q).  All ranks must call collectively with the same arguments.
 * sc_dist_lambda_max: min((1 + margin) theta, 2 max_i s_i) as sc_lambda_max.
 * sc_dist_cheb_moments: moments[0..2 order] (host) of the probes, as sc_cheb_moments.
 * sc_dist_estimate_lambda_k: dichotomy on those moments, as sc_estimate_lambda_k.
 * Errors: SC_ERR_ARG (bad sizes, plans not ranks 0..world-1, disagreeing send/receive
 * counts), SC_ERR_CUDA (CUDA or NCCL).
 */
int sc_dist_lambda_max(sc_dist* const* ds, int nheld, int iters, double margin, uint64_t seed, const int64_t* row0,
                       double* out, void* stream);
int sc_dist_cheb_moments(sc_dist* const* ds, int nheld, double lambda_max, int order, int n_probe, uint64_t seed,
                         const int64_t* row0, double* moments, void* stream);
int sc_dist_estimate_lambda_k(sc_dist* const* ds, int nheld, int k, double lambda_max, int order, int jackson,
                              int n_probe, uint64_t seed, const int64_t* row0, int max_iter, double rtol,
                              double* lambda_k, double* count_k, void* stream);

/*
 * sc_dist_kmeans -- sc_kmeans over the rows of a row partition (§4.1 step 6,
 * l.323-328; BASELINE configs[4] "full pipeline including k-means" at 8 GPUs).  The points
 * are the ranks' rows in rank-major order (rank 0's n_local[0] rows in its local order, then
 * rank 1's, ...).  Lloyd runs data-parallel: every rank assigns its own rows with the
 * single-GPU kernels; the exact fixed-point member sums and the member counts are summed over
 * the ranks as integers (order independent: the centroids are bit-identical to sc_kmeans on
 * the concatenated rows), the changed-label counts and the inertia likewise; the k-means++
 * draw is made on the global D^2 prefix in rank order (R13).
 * comms / nheld: nheld = 1 (one process per GPU, NCCL communicator from sc_comm_init; n_local
 * = this rank's count) or nheld = world (all ranks in this process, communicators from
 * sc_comm_local; one host thread per rank, reductions at a host rendezvous).
 * F[r] (device, n_local[r] x d fp32), labels[r] (device int32 [n_local[r]]) per held rank;
 * uniforms (host, restarts * k, or NULL = counter generator as sc_kmeans).  centroids (host,
 * k * d, may be NULL), inertia, iters, best_restart (host, may be NULL): equal on every rank.
 * Errors: SC_ERR_ARG (bad sizes, a rank with no rows, host buffers, total n >= 2^25),
 * SC_ERR_CUDA, SC_ERR_STATE (ranks disagreeing on the result: a bug).
 */
int sc_dist_kmeans(sc_comm* const* comms, int nheld, const float* const* F, const int64_t* n_local, int d, int k,
                   int restarts, int max_iter, uint64_t seed, const double* uniforms, int32_t* const* labels,
                   double* centroids, double* inertia, int* iters, int* best_restart, void* stream);

/* ------------------------------------------------------------------------ */
/* Row-partitioned filter with the halo exchange fused into the step kernel */
/* (north_star: "exchanges the needed rows of T_j over NVLink ... overlapped */
/* with the interior SpMM")                                */
/* ------------------------------------------------------------------------ */

typedef struct sc_p2p sc_p2p;     /* one rank's partition + peer-mapped T buffers */

/*
 * sc_p2p_create -- one rank of a row partition whose halo rows are delivered by the
 * producing rank's step kernel (NVLink peer stores from its epilogue), not by a
 * separate exchange.  g: the rank's local CSR (n_rows = n_local; columns >= n_local
 * are the halo, grouped by owner rank, ascending).  Send descriptors, CSR by local
 * row: row i is needed by peers sd_peer[e] at their halo slot sd_slot[e], e in
 * [sd_ptr[i], sd_ptr[i+1]) (sd_ptr: n_local+1 entries; sd_row[e] = i repeats the row
 * of entry e).  peer_n_local[q]: n_local of rank q.  n_global: rows of the whole
 * graph (all ranks must agree; it fixes the common column-chunk plan).  max_R:
 * widest block the partition will filter.  Arrays are copied (host or device).
 * Allocates three (n_local + n_halo) x ceil4(max_R) fp32 buffers (cudaMalloc, CUDA
 * IPC exportable) and a flag array.  world <= 8.
 */
int sc_p2p_create(sc_graph* g, int world, int rank, int64_t n_global, const int64_t* sd_ptr, const int64_t* sd_row,
                  const int32_t* sd_peer, const int64_t* sd_slot, int64_t n_desc, const int64_t* peer_n_local,
                  int max_R, sc_p2p** out);
int sc_p2p_free(sc_p2p* p);

/* sc_p2p_export -- CUDA IPC handles of the rank's three T buffers and its flag array:
 * 4 x 64 bytes written to `handles`.  sc_p2p_import -- map peer `peer`'s buffers
 * (the 256 bytes its export produced; cudaIpcOpenMemHandle, peer access enabled
 * lazily).  sc_p2p_link_local -- same for a peer created in this process (single-GPU
 * emulation and tests). */
int sc_p2p_export(sc_p2p* p, void* handles);
int sc_p2p_import(sc_p2p* p, int peer, const void* handles);
int sc_p2p_link_local(sc_p2p* p, sc_p2p* peer);

/*
 * sc_p2p_filter_f32 -- this rank's rows of Y = sum_j coeffs[j] T_j(L~) X (as
 * sc_dist_filter_f32; X, Y n_local x R in the local row order, host or device).
 * One process per GPU; every rank must make the same sequence of calls.  Before each
 * step the stream waits (one-warp kernel, acquire loads of the flags the peers
 * publish when their previous step's stores have landed; traps after ~20 s without
 * progress rather than hang).  R <= max_R.
 *
 * sc_p2p_filter_group_f32 -- all `world` ranks of a partition held by this process
 * (ps[q] has rank q, peers linked with sc_p2p_link_local), device X[q] / Y[q]: the
 * same kernels launched in a dependency order on one stream (step s of every rank,
 * then step s+1), so nothing waits: the single-GPU emulation of the fused exchange.
 */
int sc_p2p_filter_f32(sc_p2p* p, const double* coeffs, int order, double lambda_max, int R, const float* X, float* Y,
                      void* stream);
int sc_p2p_filter_group_f32(sc_p2p* const* ps, int world, const double* coeffs, int order, double lambda_max, int R,
                            const float* const* X, float* const* Y, void* stream);

/* ------------------------------------------------------------------------ */
/* Instrumentation (bench.py)                                               */
/* ------------------------------------------------------------------------ */

/*
 * sc_profile_begin / sc_profile_end -- while on, every fused-step launch is
 * bracketed by CUDA events recorded on its launching stream.  sc_profile_end
 * synchronises those events and returns: all kernels launched by the filter
 * path, fused-step launches, their summed device time (ms), and their summed
 * algorithmic bytes (CSR share + each dense operand row read/written once;
 * DESIGN.md "roofline").  Not thread-safe; profiling is process-global.
 */
int sc_profile_begin(void);
int sc_profile_end(int64_t* launches, int64_t* step_launches, double* step_ms, double* algo_bytes);

#ifdef __cplusplus
}
#endif

#endif /* SC_B200_H */
