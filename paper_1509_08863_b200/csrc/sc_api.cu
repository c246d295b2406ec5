// The C ABI (include/sc_b200.h): argument checking, host/device staging and
// dispatch to the kernels.  Every entry point cites its PAPER.md passage in the
// header.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "sc_internal.cuh"

namespace sc {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }
int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes attr;
  cudaError_t e = cudaPointerGetAttributes(&attr, p);
  if (e != cudaSuccess) {
    cudaGetLastError();   // clear sticky-less error
    return false;
  }
  return attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged;
}

int Staged::alloc(size_t b, cudaStream_t s) {
  st = s;
  keep_pool_reserved();
  cudaError_t e = cudaMallocAsync(&owned, b ? b : 1, s);
  if (e != cudaSuccess) {
    owned = nullptr;
    return fail(SC_ERR_NOMEM, std::string("cudaMallocAsync: ") + cudaGetErrorString(e));
  }
  dev = owned;
  return SC_OK;
}

int Staged::in(const void* p, size_t b, cudaStream_t s, bool copy) {
  bytes = b;
  if (is_device_ptr(p)) {
    dev = const_cast<void*>(p);
    host = nullptr;
    return SC_OK;
  }
  host = p;
  SC_TRY(alloc(b, s));
  if (copy && b) SC_CUDA_TRY(cudaMemcpyAsync(dev, p, b, cudaMemcpyHostToDevice, s));
  return SC_OK;
}

int Staged::out(void* p, cudaStream_t s) {
  if (host && bytes) {
    SC_CUDA_TRY(cudaMemcpyAsync(p, dev, bytes, cudaMemcpyDeviceToHost, s));
    SC_CUDA_TRY(cudaStreamSynchronize(s));
  }
  return SC_OK;
}

namespace {

__global__ void strengths_kernel(const int64_t* __restrict__ row_ptr, const float* __restrict__ val, int64_t n,
                                 double* __restrict__ s64, float* __restrict__ s32) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = row_ptr[i], e = row_ptr[i + 1];
    double s = 0.0;
    if (val) for (int64_t k = b; k < e; ++k) s += (double)val[k];
    else s = (double)(e - b);
    s64[i] = s;
    s32[i] = (float)s;
  }
}

__global__ void max_kernel(const double* __restrict__ v, int64_t n, unsigned long long* out) {
  double m = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = fmax(m, v[i]);
  atomicMax(out, (unsigned long long)__double_as_longlong(m));   // non-negative doubles order as integers
}

__global__ void check_csr_kernel(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col, int64_t n_rows,
                                 int64_t n_cols, int* bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_rows; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = row_ptr[i], e = row_ptr[i + 1];
    if (e < b) { atomicOr(bad, 1); continue; }
    for (int64_t k = b; k < e; ++k) {
      const int32_t c = col[k];
      if (c < 0 || c >= n_cols) atomicOr(bad, 2);
    }
  }
}

inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

int ensure_device() {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    cudaGetLastError();
    return fail(SC_ERR_CUDA, "no CUDA device available (there is no CPU fallback)");
  }
  return SC_OK;
}

}  // namespace
}  // namespace sc

using namespace sc;

namespace sc {
template <typename T>
static int filter_apply_entry(sc_graph* g, const double* coeffs, int order, double lambda_max, int R, const T* X, T* Y,
                              void* stream) {
  SC_CHECK_ARG(g && coeffs && X && Y, "null argument");
  SC_CHECK_ARG(order >= 1 && R >= 1 && lambda_max > 0.0, "order >= 1, R >= 1, lambda_max > 0 required");
  SC_CHECK_ARG(g->n_cols == g->n_rows, "sc_filter_apply needs a single-GPU graph (use sc_cheb_step)");
  SC_CHECK_ARG((const void*)X != (const void*)Y, "X and Y must not alias");
  cudaStream_t s = as_stream(stream);
  const size_t bytes = sizeof(T) * g->n_rows * R;
  Staged x, y;
  SC_TRY(x.in(X, bytes, s, true));
  SC_TRY(y.in(Y, bytes, s, false));
  SC_TRY(filter_apply<T>(g, coeffs, order, lambda_max, R, static_cast<const T*>(x.dev), static_cast<T*>(y.dev), s));
  SC_TRY(y.out(Y, s));
  return SC_OK;
}

template <typename T>
static int lowpass_entry(sc_graph* g, double lambda_c, double lambda_max, int order, int jackson, int R, uint64_t seed,
                         const T* X, T* Y, void* stream) {
  SC_CHECK_ARG(g && Y, "null argument");
  SC_CHECK_ARG(order >= 1 && R >= 1 && lambda_max > 0.0, "order >= 1, R >= 1, lambda_max > 0 required");
  SC_CHECK_ARG(g->n_cols == g->n_rows, "sc_filter_lowpass needs a single-GPU graph");
  std::vector<double> d(order + 1);
  cheby_lowpass_coeffs(lambda_c, lambda_max, order, jackson != 0, d.data());
  cudaStream_t s = as_stream(stream);
  const size_t bytes = sizeof(T) * g->n_rows * R;
  Staged x, y;
  if (X) {
    SC_TRY(x.in(X, bytes, s, true));
  } else {
    SC_TRY(x.alloc(bytes, s));
    SC_TRY(random_signals<T>(g->n_rows, R, 0, seed, 0, 1.0 / R, static_cast<T*>(x.dev), s));
  }
  SC_TRY(y.in(Y, bytes, s, false));
  SC_TRY(filter_apply<T>(g, d.data(), order, lambda_max, R, static_cast<const T*>(x.dev), static_cast<T*>(y.dev), s));
  SC_TRY(y.out(Y, s));
  return SC_OK;
}

}  // namespace sc

extern "C" {

int sc_version(void) { return 10000; }

const char* sc_last_error(void) { return sc::g_last_error.c_str(); }

int sc_graph_load(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* row_ptr, const int32_t* col_idx,
                  const float* values, sc_graph** out) {
  SC_CHECK_ARG(out, "out is NULL");
  *out = nullptr;
  SC_CHECK_ARG(n_rows >= 1 && n_cols >= n_rows && nnz >= 0, "bad sizes");
  SC_CHECK_ARG(n_cols <= INT32_MAX, "n_cols exceeds int32 column indices");
  SC_CHECK_ARG(row_ptr && (col_idx || nnz == 0), "null CSR arrays");
  SC_TRY(ensure_device());
  sc_graph* g = new sc_graph();
  auto bail = [&](int rc) { delete g; return rc; };
  g->n_rows = n_rows;
  g->n_cols = n_cols;
  g->nnz = nnz;
  g->unit_weights = values == nullptr;
  cudaGetDevice(&g->device);
  cudaDeviceGetAttribute(&g->num_sms, cudaDevAttrMultiProcessorCount, g->device);
  cudaStream_t s = 0;
  int rc;
  // CSR arrays are padded (kRowPtrPad / kColPad zeroed entries) so that the filter's 16-byte
  // aligned bulk copies of a tile's row_ptr / col_idx / values segments may over-read the tail.
  if ((rc = g->row_ptr.ensure(sizeof(int64_t) * (n_rows + 1 + kRowPtrPad))) != SC_OK) return bail(rc);
  if ((rc = g->col_idx.ensure(sizeof(int32_t) * (nnz + kColPad))) != SC_OK) return bail(rc);
  if (!g->unit_weights && (rc = g->values.ensure(sizeof(float) * (nnz + kColPad))) != SC_OK) return bail(rc);
  cudaMemsetAsync(g->row_ptr.as<int64_t>() + n_rows + 1, 0, sizeof(int64_t) * kRowPtrPad, s);
  cudaMemsetAsync(g->col_idx.as<int32_t>() + nnz, 0, sizeof(int32_t) * kColPad, s);
  if (!g->unit_weights) cudaMemsetAsync(g->values.as<float>() + nnz, 0, sizeof(float) * kColPad, s);
  if ((rc = g->strength64.ensure(sizeof(double) * n_rows)) != SC_OK) return bail(rc);
  if ((rc = g->strength32.ensure(sizeof(float) * n_rows)) != SC_OK) return bail(rc);
  auto cp = [&](void* dst, const void* src, size_t b) -> int {
    if (!b) return SC_OK;
    cudaError_t e = cudaMemcpyAsync(dst, src, b, is_device_ptr(src) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s);
    return e == cudaSuccess ? SC_OK : fail(SC_ERR_CUDA, cudaGetErrorString(e));
  };
  if ((rc = cp(g->row_ptr.ptr, row_ptr, sizeof(int64_t) * (n_rows + 1))) != SC_OK) return bail(rc);
  if ((rc = cp(g->col_idx.ptr, col_idx, sizeof(int32_t) * nnz)) != SC_OK) return bail(rc);
  if (!g->unit_weights && (rc = cp(g->values.ptr, values, sizeof(float) * nnz)) != SC_OK) return bail(rc);
  int64_t first = 0, last = 0;
  cudaMemcpy(&first, g->row_ptr.as<int64_t>(), sizeof(int64_t), cudaMemcpyDeviceToHost);
  cudaMemcpy(&last, g->row_ptr.as<int64_t>() + n_rows, sizeof(int64_t), cudaMemcpyDeviceToHost);
  if (first != 0) return bail(fail(SC_ERR_ARG, "row_ptr[0] != 0"));
  if (last != nnz) return bail(fail(SC_ERR_ARG, "row_ptr[n_rows] != nnz"));
  sc::DevBuf flag;
  if ((rc = flag.ensure(16)) != SC_OK) return bail(rc);
  cudaMemsetAsync(flag.ptr, 0, 16, s);
  check_csr_kernel<<<g->num_sms * 8, 256, 0, s>>>(g->row_ptr.as<int64_t>(), g->col_idx.as<int32_t>(), n_rows, n_cols,
                                                  flag.as<int>());
  strengths_kernel<<<g->num_sms * 8, 256, 0, s>>>(g->row_ptr.as<int64_t>(),
                                                  g->unit_weights ? nullptr : g->values.as<float>(), n_rows,
                                                  g->strength64.as<double>(), g->strength32.as<float>());
  max_kernel<<<g->num_sms * 4, 256, 0, s>>>(g->strength64.as<double>(), n_rows,
                                            reinterpret_cast<unsigned long long*>(flag.as<char>() + 8));
  int bad = 0;
  unsigned long long mx = 0;
  cudaMemcpy(&bad, flag.ptr, sizeof(int), cudaMemcpyDeviceToHost);
  cudaMemcpy(&mx, flag.as<char>() + 8, sizeof(mx), cudaMemcpyDeviceToHost);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return bail(fail(SC_ERR_CUDA, cudaGetErrorString(e)));
  if (bad & 1) return bail(fail(SC_ERR_ARG, "row_ptr is not non-decreasing"));
  if (bad & 2) return bail(fail(SC_ERR_ARG, "column index out of range [0, n_cols)"));
  double mxd;
  std::memcpy(&mxd, &mx, sizeof(double));
  g->max_strength = mxd;
  *out = g;
  return SC_OK;
}

int sc_graph_free(sc_graph* g) {
  if (g) sell_release(g);
  delete g;
  return SC_OK;
}

int sc_graph_info(const sc_graph* g, int64_t* n_rows, int64_t* n_cols, int64_t* nnz, double* max_strength) {
  SC_CHECK_ARG(g, "null graph");
  if (n_rows) *n_rows = g->n_rows;
  if (n_cols) *n_cols = g->n_cols;
  if (nnz) *nnz = g->nnz;
  if (max_strength) *max_strength = g->max_strength;
  return SC_OK;
}

int sc_graph_strengths(const sc_graph* g, double* out, void* stream) {
  SC_CHECK_ARG(g && out, "null argument");
  cudaStream_t s = as_stream(stream);
  Staged o;
  SC_TRY(o.in(out, sizeof(double) * g->n_rows, s, false));
  SC_CUDA_TRY(cudaMemcpyAsync(o.dev, g->strength64.ptr, sizeof(double) * g->n_rows, cudaMemcpyDeviceToDevice, s));
  SC_TRY(o.out(out, s));
  return SC_OK;
}

int sc_lambda_max(sc_graph* g, int iters, double margin, uint64_t seed, double* out, void* stream) {
  SC_CHECK_ARG(g && out, "null argument");
  SC_CHECK_ARG(iters >= 1 && margin >= 0.0, "iters >= 1 and margin >= 0 required");
  SC_CHECK_ARG(g->n_cols == g->n_rows, "sc_lambda_max needs a single-GPU graph");
  double theta = 0.0;
  SC_TRY(lanczos_lambda_max(g, iters, seed, &theta, as_stream(stream)));
  const double gersh = 2.0 * g->max_strength;
  double b = (1.0 + margin) * theta;
  if (!(b > 0.0) || b > gersh) b = gersh;
  if (!(b > 0.0)) b = 1.0;   // edgeless graph: any positive domain
  *out = b;
  return SC_OK;
}

int sc_cheby_coeffs(double lambda_c, double lambda_max, int order, int jackson, double* coeffs) {
  SC_CHECK_ARG(coeffs, "null coeffs");
  SC_CHECK_ARG(order >= 0 && lambda_max > 0.0, "order >= 0 and lambda_max > 0 required");
  cheby_lowpass_coeffs(lambda_c, lambda_max, order, jackson != 0, coeffs);
  return SC_OK;
}

int sc_filter_order(double ratio, double delta, int jackson, double theta, int n_grid, int m_max, int* m_star,
                    double* err, void* stream) {
  SC_CHECK_ARG(m_star, "null m_star");
  SC_CHECK_ARG(ratio > 0.0 && ratio <= 1.0 && delta > 0.0 && theta >= 0.0 && theta < 1.0,
               "0 < ratio <= 1, delta > 0, 0 <= theta < 1 required");
  SC_CHECK_ARG(n_grid >= 2 && n_grid <= (1 << 24) && m_max >= 1 && m_max <= 4096,
               "2 <= n_grid <= 2^24 and 1 <= m_max <= 4096 required");
  return filter_order(ratio, delta, jackson != 0, theta, n_grid, m_max, m_star, err, as_stream(stream));
}

static int random_common_check(int64_t n, int R) {
  SC_CHECK_ARG(n >= 0 && R >= 1, "n >= 0 and R >= 1 required");
  return ensure_device();
}

int sc_random_signals_f32(int64_t n, int R, int64_t row0, uint64_t seed, int stream_id, double variance, float* out,
                          void* stream) {
  SC_TRY(random_common_check(n, R));
  SC_CHECK_ARG(out || n == 0, "null out");
  if (n == 0) return SC_OK;
  cudaStream_t s = as_stream(stream);
  Staged o;
  SC_TRY(o.in(out, sizeof(float) * n * R, s, false));
  SC_TRY(random_signals<float>(n, R, row0, seed, stream_id, variance, static_cast<float*>(o.dev), s));
  SC_TRY(o.out(out, s));
  return SC_OK;
}

int sc_random_signals_f64(int64_t n, int R, int64_t row0, uint64_t seed, int stream_id, double variance, double* out,
                          void* stream) {
  SC_TRY(random_common_check(n, R));
  SC_CHECK_ARG(out || n == 0, "null out");
  if (n == 0) return SC_OK;
  cudaStream_t s = as_stream(stream);
  Staged o;
  SC_TRY(o.in(out, sizeof(double) * n * R, s, false));
  SC_TRY(random_signals<double>(n, R, row0, seed, stream_id, variance, static_cast<double*>(o.dev), s));
  SC_TRY(o.out(out, s));
  return SC_OK;
}

int sc_filter_apply_f32(sc_graph* g, const double* coeffs, int order, double lambda_max, int R, const float* X,
                        float* Y, void* stream) {
  return filter_apply_entry<float>(g, coeffs, order, lambda_max, R, X, Y, stream);
}

int sc_filter_apply_f64(sc_graph* g, const double* coeffs, int order, double lambda_max, int R, const double* X,
                        double* Y, void* stream) {
  return filter_apply_entry<double>(g, coeffs, order, lambda_max, R, X, Y, stream);
}

int sc_filter_lowpass_f32(sc_graph* g, double lambda_c, double lambda_max, int order, int jackson, int R,
                          uint64_t seed, const float* X, float* Y, void* stream) {
  return lowpass_entry<float>(g, lambda_c, lambda_max, order, jackson, R, seed, X, Y, stream);
}

int sc_filter_lowpass_f64(sc_graph* g, double lambda_c, double lambda_max, int order, int jackson, int R,
                          uint64_t seed, const double* X, double* Y, void* stream) {
  return lowpass_entry<double>(g, lambda_c, lambda_max, order, jackson, R, seed, X, Y, stream);
}

int sc_cheb_step_f32(sc_graph* g, int64_t row_begin, int64_t row_end, int R, const float* T_prev, int64_t ld_prev,
                     const float* T_cur, int64_t ld_cur, float* T_next, int64_t ld_next, float* Y, int64_t ld_y,
                     double a, double b_cur, double b_prev, double cy_prev, double cy_cur, double cy_next,
                     int y_mode, void* stream) {
  SC_CHECK_ARG(g && T_cur, "null argument");
  SC_CHECK_ARG(0 <= row_begin && row_begin <= row_end && row_end <= g->n_rows, "bad row range");
  SC_CHECK_ARG(y_mode >= 0 && y_mode <= 2 && (y_mode == 0 || Y), "bad y_mode / Y");
  SC_CHECK_ARG(T_prev || (b_prev == 0.0 && cy_prev == 0.0), "T_prev required");
  SC_CHECK_ARG(R % 4 == 0 && ld_cur % 4 == 0 && (!T_prev || ld_prev % 4 == 0) && (!T_next || ld_next % 4 == 0) &&
                   (!Y || ld_y % 4 == 0),
               "sc_cheb_step_f32 needs R and strides that are multiples of 4");
  cudaStream_t s = as_stream(stream);
  // chunk the R columns into supported widths (<= 128)
  int col0 = 0;
  while (col0 < R) {
    int w = 128;
    while (w > R - col0) w >>= 1;
    StepParams p{};
    p.row_begin = row_begin;
    p.row_end = row_end;
    p.width = w;
    p.tprev = T_prev ? T_prev + col0 : nullptr;
    p.ld_prev = ld_prev;
    p.tcur = T_cur + col0;
    p.ld_cur = ld_cur;
    p.tnext = T_next ? T_next + col0 : nullptr;
    p.ld_next = ld_next;
    p.y = Y ? Y + col0 : nullptr;
    p.ld_y = ld_y;
    p.a = a;
    p.b_cur = b_cur;
    p.b_prev = b_prev;
    p.cy_prev = cy_prev;
    p.cy_cur = cy_cur;
    p.cy_next = cy_next;
    p.y_mode = y_mode;
    SC_TRY(launch_step<float>(g, p, s));
    col0 += w;
  }
  return SC_OK;
}

int sc_cheb_moments(sc_graph* g, double lambda_max, int order, int R, uint64_t seed, const double* X, double* moments,
                    void* stream) {
  SC_CHECK_ARG(g && moments, "null argument");
  SC_CHECK_ARG(order >= 1 && R >= 1 && lambda_max > 0.0, "order >= 1, R >= 1, lambda_max > 0 required");
  SC_CHECK_ARG(g->n_cols == g->n_rows, "sc_cheb_moments needs a single-GPU graph");
  cudaStream_t s = as_stream(stream);
  const size_t bytes = sizeof(double) * g->n_rows * R;
  Staged x;
  if (X) {
    SC_TRY(x.in(X, bytes, s, true));
  } else {
    SC_TRY(x.alloc(bytes, s));
    SC_TRY(random_signals<double>(g->n_rows, R, 0, seed, 2, 1.0 / R, static_cast<double*>(x.dev), s));
  }
  std::vector<double> mu;
  SC_TRY(cheb_moments(g, lambda_max, order, R, static_cast<const double*>(x.dev), mu, s));
  if (is_device_ptr(moments)) {
    SC_CUDA_TRY(cudaMemcpyAsync(moments, mu.data(), sizeof(double) * mu.size(), cudaMemcpyHostToDevice, s));
    SC_CUDA_TRY(cudaStreamSynchronize(s));
  } else {
    std::memcpy(moments, mu.data(), sizeof(double) * mu.size());
  }
  return SC_OK;
}

int sc_eigencount_from_moments(const double* moments, int order, double lambda_c, double lambda_max, int jackson,
                               double* count) {
  SC_CHECK_ARG(moments && count, "null argument");
  SC_CHECK_ARG(order >= 1 && lambda_max > 0.0, "order >= 1 and lambda_max > 0 required");
  std::vector<double> d(order + 1);
  cheby_lowpass_coeffs(lambda_c, lambda_max, order, jackson != 0, d.data());
  *count = count_from_moments(moments, order, d.data());
  return SC_OK;
}

int sc_lambda_k_from_moments(const double* moments, int order, int k, double lambda_max, int jackson, int max_iter,
                             double rtol, double* lambda_k, double* count_k) {
  SC_CHECK_ARG(moments && lambda_k && count_k, "null argument");
  SC_CHECK_ARG(order >= 1 && k >= 1 && max_iter >= 1 && rtol > 0.0 && lambda_max > 0.0, "bad arguments");
  return lambda_k_dichotomy(moments, order, k, lambda_max, jackson != 0, max_iter, rtol, lambda_k, count_k);
}

int sc_estimate_lambda_k(sc_graph* g, int k, double lambda_max, int order, int jackson, int n_probe, uint64_t seed,
                         int max_iter, double rtol, double* lambda_k, double* count_k, void* stream) {
  SC_CHECK_ARG(g && lambda_k && count_k, "null argument");
  SC_CHECK_ARG(k >= 1 && k < g->n_rows && n_probe >= 1 && order >= 1 && max_iter >= 1 && rtol > 0.0,
               "bad arguments");
  std::vector<double> mu((size_t)2 * order + 1);
  SC_TRY(sc_cheb_moments(g, lambda_max, order, n_probe, seed, nullptr, mu.data(), stream));
  return lambda_k_dichotomy(mu.data(), order, k, lambda_max, jackson != 0, max_iter, rtol, lambda_k, count_k);
}

int sc_normalize_rows_f32(float* F, int64_t n, int d, void* stream) {
  SC_CHECK_ARG(F && n >= 0 && d >= 1, "bad arguments");
  SC_TRY(ensure_device());
  if (n == 0) return SC_OK;
  cudaStream_t s = as_stream(stream);
  Staged f;
  SC_TRY(f.in(F, sizeof(float) * n * d, s, true));
  SC_TRY(normalize_rows_f32(static_cast<float*>(f.dev), n, d, s));
  SC_TRY(f.out(F, s));
  return SC_OK;
}

int sc_kmeans(const float* F, int64_t n, int d, int k, int restarts, int max_iter, uint64_t seed,
              const double* uniforms, int32_t* labels, double* centroids, double* inertia, int* iters,
              int* best_restart, void* stream) {
  SC_CHECK_ARG(F && labels, "null argument");
  SC_CHECK_ARG(n >= 1 && d >= 1 && k >= 1 && k <= n && restarts >= 1 && max_iter >= 1, "bad arguments");
  SC_CHECK_ARG(n < (int64_t(1) << 25), "n must be < 2^25 for the exact centroid accumulator");
  SC_TRY(ensure_device());
  cudaStream_t s = as_stream(stream);
  Staged f, l;
  SC_TRY(f.in(F, sizeof(float) * n * d, s, true));
  SC_TRY(l.in(labels, sizeof(int32_t) * n, s, false));
  std::vector<double> u;
  const double* uh = nullptr;
  if (uniforms) {
    u.resize((size_t)restarts * k);
    if (is_device_ptr(uniforms)) {
      SC_CUDA_TRY(cudaMemcpyAsync(u.data(), uniforms, sizeof(double) * u.size(), cudaMemcpyDeviceToHost, s));
      SC_CUDA_TRY(cudaStreamSynchronize(s));
    } else {
      std::memcpy(u.data(), uniforms, sizeof(double) * u.size());
    }
    uh = u.data();
  }
  std::vector<double> C(centroids ? (size_t)k * d : 0);
  SC_TRY(kmeans_run(static_cast<const float*>(f.dev), n, d, k, restarts, max_iter, seed, uh,
                    static_cast<int32_t*>(l.dev), centroids ? C.data() : nullptr, inertia, iters, best_restart, s));
  SC_TRY(l.out(labels, s));
  if (centroids) {
    if (is_device_ptr(centroids)) {
      SC_CUDA_TRY(cudaMemcpyAsync(centroids, C.data(), sizeof(double) * C.size(), cudaMemcpyHostToDevice, s));
      SC_CUDA_TRY(cudaStreamSynchronize(s));
    } else {
      std::memcpy(centroids, C.data(), sizeof(double) * C.size());
    }
  }
  SC_CUDA_TRY(cudaStreamSynchronize(s));
  return SC_OK;
}

int sc_ari(const int32_t* a, const int32_t* b, int64_t n, double* out, void* stream) {
  SC_CHECK_ARG(a && b && out && n >= 1, "bad arguments");
  SC_TRY(ensure_device());
  cudaStream_t s = as_stream(stream);
  Staged sa, sb;
  SC_TRY(sa.in(a, sizeof(int32_t) * n, s, true));
  SC_TRY(sb.in(b, sizeof(int32_t) * n, s, true));
  return ari_dev(static_cast<const int32_t*>(sa.dev), static_cast<const int32_t*>(sb.dev), n, out, s);
}

int sc_stability(sc_graph* g, int k_min, int k_max, int J, int R, int order, int jackson, int n_probe, uint64_t seed,
                 int restarts, int max_iter, double lambda_max, const double* lambda_k, double* gamma,
                 double* lambda_k_out, int32_t* labels, void* stream) {
  SC_CHECK_ARG(g && gamma, "null argument");
  SC_CHECK_ARG(1 <= k_min && k_min <= k_max && k_max < g->n_rows, "1 <= k_min <= k_max < n required");
  SC_CHECK_ARG(J >= 2 && R >= 1 && order >= 1 && restarts >= 1 && max_iter >= 1 && (lambda_k || n_probe >= 1),
               "J >= 2, R, order, restarts, max_iter, n_probe >= 1 required");
  SC_CHECK_ARG(g->n_cols == g->n_rows, "sc_stability needs a single-GPU graph");
  SC_CHECK_ARG(g->n_rows < (int64_t(1) << 25), "n must be < 2^25 for the exact centroid accumulator");
  cudaStream_t s = as_stream(stream);
  const int K = k_max - k_min + 1;
  Staged lab;
  const size_t lbytes = sizeof(int32_t) * (size_t)K * J * g->n_rows;
  if (labels) {
    SC_TRY(lab.in(labels, lbytes, s, false));
  } else {
    SC_TRY(lab.alloc(lbytes, s));
  }
  SC_TRY(stability_scan(g, k_min, k_max, J, R, order, jackson != 0, n_probe, seed, restarts, max_iter, lambda_max,
                        lambda_k, gamma, lambda_k_out, static_cast<int32_t*>(lab.dev), s));
  if (labels) SC_TRY(lab.out(labels, s));
  SC_CUDA_TRY(cudaStreamSynchronize(s));
  return SC_OK;
}

int sc_profile_begin(void) {
  profile_begin();
  return SC_OK;
}

int sc_profile_end(int64_t* launches, int64_t* step_launches, double* step_ms, double* algo_bytes) {
  return profile_end(launches, step_launches, step_ms, algo_bytes);
}

// m* selection inside sc_cluster (order < 0): PAPER.md l.162 fixes delta = 0.1; the band and grid are
// DESIGN.md reading R18's
static constexpr double kOrderDelta = 0.1, kOrderTheta = 0.1;
static constexpr int kOrderGrid = 10000, kOrderMax = 2000;

int sc_cluster(sc_graph* g, int k, int R, int order, int jackson, int n_probe, uint64_t seed, int restarts,
               int max_iter, int normalize, int32_t* labels, double* info, void* stream) {
  SC_CHECK_ARG(g && labels, "null argument");
  SC_CHECK_ARG(k >= 1 && k < g->n_rows && R >= 1 && order != 0 && n_probe >= 1 && restarts >= 1 && max_iter >= 1,
               "bad arguments");
  // order < 0: step 2 at order -order, step 3's m = m*(lambda~_k/lambda_N; delta = 0.1)
  const int est_order = order > 0 ? order : -order;
  cudaStream_t s = as_stream(stream);
  // env SC_CLUSTER_TRACE: per-phase device-synchronised times on stderr (tooling)
  const bool trace = std::getenv("SC_CLUSTER_TRACE") != nullptr;
  double t_ph[4] = {0, 0, 0, 0};
  auto t_now = [] { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
  double t_mark = 0.0;
  auto phase = [&](int i) -> int {
    if (!trace) return SC_OK;
    SC_CUDA_TRY(cudaStreamSynchronize(s));
    const double t = t_now();
    if (i >= 0) t_ph[i] = t - t_mark;
    t_mark = t;
    return SC_OK;
  };
  SC_TRY(phase(-1));
  double lmax = 0.0, lk = 0.0, ck = 0.0;
  SC_TRY(sc_lambda_max(g, 60, 0.01, seed ^ 0x1a2b3c4dULL, &lmax, stream));
  SC_TRY(phase(0));
  SC_TRY(sc_estimate_lambda_k(g, k, lmax, est_order, 1, n_probe, seed ^ 0x5e5e5e5eULL, 40, 1e-4, &lk, &ck, stream));
  int filt_order = order;
  if (order < 0) {
    SC_TRY(filter_order(std::min(1.0, lk / lmax), kOrderDelta, jackson != 0, kOrderTheta, kOrderGrid, kOrderMax,
                        &filt_order, nullptr, s));
    if (filt_order == 0) filt_order = kOrderMax;
  }
  SC_TRY(phase(1));
  DevBuf feats;
  SC_TRY(feats.ensure(sizeof(float) * g->n_rows * R));
  SC_TRY(sc_filter_lowpass_f32(g, lk, lmax, filt_order, jackson, R, seed, nullptr, feats.as<float>(), stream));
  if (normalize) SC_TRY(normalize_rows_f32(feats.as<float>(), g->n_rows, R, s));
  SC_TRY(phase(2));
  double inertia = 0.0;
  int it = 0, best = 0;
  SC_TRY(sc_kmeans(feats.as<float>(), g->n_rows, R, k, restarts, max_iter, seed, nullptr, labels, nullptr, &inertia,
                   &it, &best, stream));
  SC_TRY(phase(3));
  if (trace)
    std::fprintf(stderr, "[sc_cluster] lambda_max %.4f s, lambda_k %.4f s, filter %.4f s, k-means %.4f s\n", t_ph[0],
                 t_ph[1], t_ph[2], t_ph[3]);
  if (info) {
    info[0] = lmax;
    info[1] = lk;
    info[2] = ck;
    info[3] = inertia;
    info[4] = it;
    info[5] = best;
    info[6] = filt_order;
  }
  return SC_OK;
}

}  // extern "C"
