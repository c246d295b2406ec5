// Internal declarations shared by the CUDA translation units of libsc_b200.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "sc_b200.h"

namespace sc {

// ---------------------------------------------------------------------------
// error plumbing
// ---------------------------------------------------------------------------
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);

struct Status {
  int code = SC_OK;
};

#define SC_CUDA_TRY(expr)                                                         \
  do {                                                                            \
    cudaError_t _e = (expr);                                                      \
    if (_e != cudaSuccess)                                                        \
      return ::sc::fail(SC_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)

#define SC_TRY(expr)                \
  do {                              \
    int _rc = (expr);               \
    if (_rc != SC_OK) return _rc;   \
  } while (0)

#define SC_CHECK_ARG(cond, msg) \
  do {                          \
    if (!(cond)) return ::sc::fail(SC_ERR_ARG, msg); \
  } while (0)

// ---------------------------------------------------------------------------
// device buffers
// ---------------------------------------------------------------------------
struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
  }
  int ensure(size_t b) {   // grow-only
    if (b <= bytes) return SC_OK;
    release();
    if (b == 0) return SC_OK;
    cudaError_t e = cudaMalloc(&ptr, b);
    if (e != cudaSuccess) { ptr = nullptr; return fail(SC_ERR_NOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e)); }
    bytes = b;
    return SC_OK;
  }
  template <typename T> T* as() const { return static_cast<T*>(ptr); }
};

// Stream-ordered scratch buffer (cudaMallocAsync / cudaFreeAsync on its stream): no
// device-wide synchronisation, so concurrent streams (sc_stability's k-means workers)
// stay concurrent.
// The stream-ordered pool of the current device keeps up to 8 GB of freed memory reserved
// (default: 0, i.e. trimmed at every synchronisation, so each call re-maps its workspaces --
// measured as sporadic 0.2-0.9 s host stalls on repeated calls).  Idempotent, cheap.
inline void keep_pool_reserved() {
  static std::once_flag once[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return;
  std::call_once(once[dev], [dev] {   // worker threads may get here concurrently
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = 8ull << 30;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  });
}

struct PoolBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  cudaStream_t st = 0;
  PoolBuf() = default;
  PoolBuf(const PoolBuf&) = delete;
  PoolBuf& operator=(const PoolBuf&) = delete;
  ~PoolBuf() { release(); }
  void release() {   // before the owning stream is destroyed
    if (ptr) cudaFreeAsync(ptr, st);
    ptr = nullptr;
    bytes = 0;
  }
  int ensure(size_t b, cudaStream_t s) {
    if (b <= bytes && ptr) return SC_OK;
    if (ptr) cudaFreeAsync(ptr, st);
    ptr = nullptr;
    bytes = 0;
    st = s;
    keep_pool_reserved();
    cudaError_t e = cudaMallocAsync(&ptr, b ? b : 1, s);
    if (e != cudaSuccess) { ptr = nullptr; return fail(SC_ERR_NOMEM, std::string("cudaMallocAsync: ") + cudaGetErrorString(e)); }
    bytes = b;
    return SC_OK;
  }
  template <typename T> T* as() const { return static_cast<T*>(ptr); }
};

// Is p a device (or managed) pointer of the current device?
bool is_device_ptr(const void* p);

// Host<->device staging for an argument that may be host or device memory.
// Owned staging memory comes from the stream-ordered pool (cudaMallocAsync), so
// repeated host-buffer calls do not pay cudaMalloc/cudaFree.
struct Staged {
  void* dev = nullptr;          // device view
  const void* host = nullptr;   // original host pointer (if staged)
  size_t bytes = 0;
  void* owned = nullptr;
  cudaStream_t st = 0;
  Staged() = default;
  Staged(const Staged&) = delete;
  Staged& operator=(const Staged&) = delete;
  ~Staged() {
    if (owned) cudaFreeAsync(owned, st);
  }
  int alloc(size_t b, cudaStream_t s);                           // owned device buffer
  int in(const void* p, size_t b, cudaStream_t s, bool copy);   // stage to device
  int out(void* p, cudaStream_t s);                               // copy back if host
};

// ---------------------------------------------------------------------------
// graph handle
// ---------------------------------------------------------------------------
}  // namespace sc

namespace sc {
constexpr int kRowPtrPad = 8;   // extra zeroed row_ptr entries past n_rows+1
constexpr int kColPad = 8;      // extra zeroed col_idx / values entries past nnz
}  // namespace sc

struct sc_graph {
  int64_t n_rows = 0, n_cols = 0, nnz = 0;
  bool unit_weights = true;
  double max_strength = 0.0;
  sc::DevBuf row_ptr;     // int64 [n_rows+1]
  sc::DevBuf col_idx;     // int32 [nnz]
  sc::DevBuf values;      // float [nnz] (empty if unit weights)
  sc::DevBuf strength64;  // double [n_rows]
  sc::DevBuf strength32;  // float  [n_rows]
  // workspace (grow-only)
  sc::DevBuf ws_a, ws_b, ws_sig, ws_part, ws_misc, ws_split, ws_limbs;
  // per (tile rows, row_begin, row_end): degree-sorted row order inside each tile (uint16)
  mutable std::map<std::tuple<int, int64_t, int64_t>, std::unique_ptr<sc::DevBuf>> tile_orders;
  mutable std::mutex tile_orders_mu;
  // resident-CSR small-graph plans per (chunk width, element size): host ints
  // {usable, grid, cap_rows, cap_nnz, smem}, device tile ranges, step coefficients
  std::map<std::pair<int, int>, std::vector<int64_t>> resident_plans;
  std::map<std::pair<int, int>, std::unique_ptr<sc::DevBuf>> resident_tiles;
  sc::DevBuf resident_coef;
  // filter_apply's structural chunk-width choice (key (0, 0): 1 = 64-column chunks)
  std::map<std::pair<int, int>, int> chunk_tuned;
  std::mutex chunk_tuned_mu;
  // dynamic tile scheduling of the step kernel: one tile counter per launch from a ring of
  // kTileCtrRing slots, zeroed once; the last tile request of a launch resets its slot
  mutable sc::DevBuf tile_ctr_ring;
  mutable int64_t tile_ctr_seq = 0;
  mutable std::mutex tile_ctr_mu;
  int num_sms = 148;
  int device = 0;
};

namespace sc {

// ---------------------------------------------------------------------------
// kernels / drivers (defined in the .cu files)
// ---------------------------------------------------------------------------
// Fused peer-to-peer halo exchange (sc_p2p.cu): device-side description of where a rank's
// boundary rows go.  Row i of this rank is needed by the peers listed in
// [sd_ptr[i], sd_ptr[i+1]): peer sd_peer[e] keeps it at halo slot sd_slot[e], i.e. row
// peer_nl[q] + sd_slot[e] of its buffers.  peer_buf[b][q] is peer q's T buffer b (b = 0, 1, 2)
// mapped into this process (NVLink peer memory via CUDA IPC, or local memory in the
// single-GPU emulation); peer_flags[q] is peer q's flag array ([world] int64, written by
// rank r at index r).
struct P2PDev {
  const int64_t* sd_ptr;
  const int32_t* sd_peer;
  const int64_t* sd_slot;
  const int64_t* peer_nl;
  void* peer_buf[3][8];
  int64_t* peer_flags[8];
  unsigned* done_ctr;
  int64_t row0;      // rows below row0 have no descriptors (interior rows)
  int rank, world;
};
constexpr int kP2PMaxWorld = 8;

struct StepParams {
  int64_t row_begin, row_end;
  const void* tprev; int64_t ld_prev;
  const void* tcur;  int64_t ld_cur;
  void* tnext;       int64_t ld_next;
  void* y;           int64_t ld_y;
  double a, b_cur, b_prev;
  double cy_prev, cy_cur, cy_next;
  int y_mode;        // 0 none, 1 write, 2 accumulate
  int width;         // columns processed (chunk width)
  int total_width;   // all columns of the block (for the profiler's CSR share)
  // moments mode (fp64 only): per-block partial sums written to `part`
  double* part;      // [gridDim.x][3] : <Tc,Tc>, <Tn,Tc>, <Tn,Tn>
  // moments on the SELL kernel (fp64): the three sums as exact fixed-point integers (value
  // x 2^80, four 32-bit limbs each accumulated in a uint64 -- order independent), [3][4]
  unsigned long long* mom_limbs;
  // fused exchange (nullptr: none): T_{s+1} rows also stored into the peers' buffer
  // p2p_next; after the launch the last CTA publishes p2p_signal in every peer's flags
  const P2PDev* p2p;
  int p2p_next;
  int64_t p2p_signal;
  // dynamic tile scheduling (nullptr: static round-robin): tiles are taken from this counter
  unsigned* tile_ctr;
  // L2 eviction policies of the dense streams (experiment knob SC_L2POL, 0 = default):
  // bits 0-1 own row T_s[i] (0 evict_first, 1 evict_normal, 2 evict_last),
  // bits 2-3 T_{s+1} store (0 no hint, 1 evict_first, 2 evict_last, 3 evict_normal),
  // bits 4-5 T_{s-1} row (0 evict_first, 1 evict_normal)
  unsigned l2pol;
  // split gather (SELL path): 0 none; 1 = columns [0, split_col) only, the row
  // sums go to split_buf (row stride width) and there is no epilogue; 2 = columns
  // [split_col, n_cols), split_buf added before the epilogue
  int split_mode;
  int64_t split_col;
  void* split_buf;
};

// launch one fused step for `width` columns starting at the given pointers
template <typename T>
int launch_step(const sc_graph* g, const StepParams& p, cudaStream_t s);

// one fused step over the sliced padded CSR (sc_sell.cu); T_s needs a zero row at n_cols.
// *algo_bytes (optional): the step's algorithmic bytes
template <typename T>
int launch_sell_step(const sc_graph* g, const StepParams& p, cudaStream_t s, double* algo_bytes);
bool sell_enabled();                       // env SC_SELL (default 1)
template <typename T>
int sell_usable(const sc_graph* g, int width, int64_t row_begin, int64_t row_end, cudaStream_t s, bool* ok,
                int64_t split_col = 0);
int64_t sell_split_col(const sc_graph* g, int width, size_t elem);   // 0: no split gather
void sell_release(const sc_graph* g);      // drop the graph's cached SELL plans
int64_t max_row_degree(const sc_graph* g, int64_t r0, int64_t r1, cudaStream_t s);
bool dyn_tiles_on();                       // env SC_DYN_TILES (default 1)
unsigned* next_tile_ctr(const sc_graph* g, cudaStream_t s);   // a self-resetting tile counter slot
// one fused step of the row-partitioned paths: the SELL kernel when it can run this chunk width
// and row range (the caller keeps row n_cols of p.tcur, stride p.ld_cur, zero), else the
// plain-CSR kernel; fused-exchange epilogue (p.p2p) on either
template <typename T>
int launch_step_any(const sc_graph* g, StepParams p, cudaStream_t s);

// degree-sorted row order of every tile of tr rows over [row_begin, row_end) (cached on g)
const uint16_t* tile_order(const sc_graph* g, int tr, int64_t row_begin, int64_t row_end, cudaStream_t s);

// launch profiler hooks for kernels launched outside launch_step (one launch = `steps` steps)
void prof_launch_begin(cudaStream_t s, cudaEvent_t* e0);
void prof_launch_end(cudaStream_t s, cudaEvent_t e0, double algo_bytes, int steps);

// all `order` steps of one column chunk in one cooperative launch when the CSR fits the
// aggregate shared memory; *ok = false otherwise (sc_resident.cu)
// stack != nullptr: stack mode (every T_j kept at stack + j * slot, row stride ld_x, T_0 in slot
// 0, no Y) -- sc_stability's recurrence
template <typename T>
int resident_filter(sc_graph* g, const double* d, int order, double lambda_max, int w, const T* Xc, int64_t ld_x,
                    T* Yc, int64_t ld_y, T* buf0, T* buf1, cudaStream_t s, bool* ok, T* stack = nullptr,
                    int64_t slot = 0);

// column chunk widths (each a supported kernel width) covering R columns
template <typename T>
std::vector<int> chunk_widths(int R, int64_t n_cols);

// full filter: Y = sum_j coeffs_j T_j X   (X, Y device, row-major n x R)
template <typename T>
int filter_apply(sc_graph* g, const double* coeffs, int order, double lambda_max, int R,
                 const T* X, T* Y, cudaStream_t s);

// launch profiler
void profile_begin();
int profile_end(int64_t* launches, int64_t* step_launches, double* step_ms, double* algo_bytes);

// Chebyshev moments (fp64) into host vector
int cheb_moments(sc_graph* g, double lambda_max, int order, int R, const double* X,
                 std::vector<double>& mu, cudaStream_t s);

// random signals on device
template <typename T>
int random_signals(int64_t n, int R, int64_t row0, uint64_t seed, int stream_id, double variance,
                   T* out, cudaStream_t s);

// Lanczos
int lanczos_lambda_max(sc_graph* g, int iters, uint64_t seed, double* theta, cudaStream_t s);
// its building blocks (sc_linalg.cu), for the row-partitioned version (sc_dist.cu):
// w = L v - beta_j vprev over g's rows (v has g->n_cols entries: local rows + halo)
namespace lz {
constexpr int kDotBlocks = 296;   // partials per dot product (part must hold this many)
int spmv(const sc_graph* g, const double* v, const double* vprev, const double* beta_j, double* w, cudaStream_t s);
int dot_local(const double* a, const double* b, int64_t n, double* part, double* out, cudaStream_t s);
int axpy_neg(double* w, const double* v, const double* alpha, int64_t n, cudaStream_t s);
int scale_inv_sqrt(double* out, const double* w, const double* b2, double* beta, int64_t n, cudaStream_t s);
double theta_from(const std::vector<double>& alpha, const std::vector<double>& beta);
}  // namespace lz

// one fused step in MOMENTS mode (fp64, static tile schedule): per-CTA partial sums of
// <T_s,T_s>, <T_{s+1},T_s>, <T_{s+1},T_{s+1}> into p.part[grid][3]; *grid = CTAs launched
int launch_moments_step(const sc_graph* g, const StepParams& p, cudaStream_t s, int* grid);
// out[0..2] = sum of the grid partials, fixed order
int reduce_moment_partials(const double* part, int grid, double* out, cudaStream_t s);

// host math (sc_host.cpp)
void cheby_lowpass_coeffs(double lambda_c, double lambda_max, int order, bool jackson, double* out);
// m*(ratio; delta) on the device (sc_order.cu); *m_star = 0 if no order <= m_max meets delta
int filter_order(double ratio, double delta, bool jackson, double theta, int n_grid, int m_max, int* m_star,
                 double* err_out, cudaStream_t s);
double count_from_moments(const double* mu, int order, const double* d);
int lambda_k_dichotomy(const double* mu, int order, int k, double lambda_max, bool jackson,
                       int max_iter, double rtol, double* lambda_k, double* count_k);
double tridiag_max_eig(const std::vector<double>& alpha, const std::vector<double>& beta);

// k-means and friends
int normalize_rows_f32(float* F, int64_t n, int d, cudaStream_t s);

// Collective operations of one rank of a row partition (the distributed k-means): in-place
// reductions of device buffers over the ranks, ordered on stream s.  Implementations: NCCL
// (one process per GPU, sc_dist.cu) and the single-process emulation (one host thread per
// rank on one GPU, host-side rendezvous: no kernel ever waits for another rank).
struct Coll {
  int rank = 0, world = 1;
  virtual ~Coll() = default;
  virtual int sum_u64(unsigned long long* p, size_t n, cudaStream_t s) = 0;   // wrap-around integer sums
  virtual int sum_u32(unsigned* p, size_t n, cudaStream_t s) = 0;
  virtual int sum_i32(int* p, size_t n, cudaStream_t s) = 0;
  virtual int sum_f64(double* p, size_t n, cudaStream_t s) = 0;
  virtual int max_u32(unsigned* p, size_t n, cudaStream_t s) = 0;
};

// tcgen05 assignment screen (sc_kmeans_tc.cu): the points (all, or the pruning list) grouped
// by their current label, screened in centred coordinates on the tensor cores with a rigorous
// bound; decided points get label / exact dmin / lo, the rest go to amb for the exact scan
struct TcWork {
  PoolBuf cnt, off, items, gperm, panels, pscal, fix;
};
bool tc_screen_supported(int k, int d);
int tc_screen(const float* F, int64_t n, int d, const double* C, const float* Cf, const double* cm, int k,
              const int32_t* old_lab, const int32_t* list, const int* list_len, int32_t* lab, double* dmin,
              double* lo, int32_t* amb, int* amb_len, TcWork& w, cudaStream_t s);

// k-means over the rows of every rank (distributed Lloyd): the points are the
// ranks' local rows in rank-major order (rank 0's n_0 rows, then rank 1's ...); row_off = this
// rank's first global index, n_global = all ranks' rows.  Every rank returns the same
// centroids / inertia / iterations / restart and its own labels.
int kmeans_run_dist(const float* F, int64_t n_local, int64_t row_off, int64_t n_global, int d, int k, int restarts,
                    int max_iter, uint64_t seed, const double* uniforms_host, int32_t* labels_dev,
                    double* centroids_host, double* inertia, int* iters, int* best_restart, Coll* coll,
                    cudaStream_t s);
// max_workers: concurrent restarts (0: env SC_KMEANS_WORKERS, default 10 -- all of a
// 10-restart call; callers that already run several k-means problems at once pass fewer)
int kmeans_run(const float* F, int64_t n, int d, int k, int restarts, int max_iter,
               uint64_t seed, const double* uniforms_host, int32_t* labels_dev,
               double* centroids_host, double* inertia, int* iters, int* best_restart,
               cudaStream_t s, int max_workers = 0);
int ari_dev(const int32_t* a, const int32_t* b, int64_t n, double* out, cudaStream_t s);

// stability measure gamma(k) over [k_min, k_max] (sc_stability.cu)
int stability_scan(sc_graph* g, int k_min, int k_max, int J, int R, int order, bool jackson, int n_probe,
                   uint64_t seed, int restarts, int max_iter, double lambda_max, const double* lambda_k_in,
                   double* gamma, double* lambda_k_out, int32_t* labels_dev, cudaStream_t s);

// counter-based RNG (host side, identical to the device one)
uint64_t splitmix64_host(uint64_t x);
double uniform_host(uint64_t seed, int stream_id, uint64_t ctr);

}  // namespace sc
