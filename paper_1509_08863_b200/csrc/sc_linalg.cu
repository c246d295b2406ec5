// Random signals (counter-based), strengths, and the Lanczos bound of lambda_N.
//
// PAPER.md §3.1 lines 182-185 / §4.1 step 4: R has i.i.d. N(0, 1/eta) entries.
// PAPER.md §4.1 step 1 (line 309): "Estimate [trefethen] L's largest eigenvalue".
#include <cmath>

#include "sc_internal.cuh"

namespace sc {

// ---------------------------------------------------------------------------
// counter-based generator (same definition as scinputs/signals.py)
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t splitmix64_hd(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

static const uint64_t kSalt[3] = {0x0ULL, 0xA5A5A5A5A5A5A5A5ULL, 0x5BD1E9955BD1E995ULL};

uint64_t splitmix64_host(uint64_t x) { return splitmix64_hd(x); }

static uint64_t stream_key(uint64_t seed, int stream_id) {
  return splitmix64_hd(seed ^ kSalt[stream_id < 0 || stream_id > 2 ? 0 : stream_id]);
}

double uniform_host(uint64_t seed, int stream_id, uint64_t ctr) {
  const uint64_t h = splitmix64_hd(stream_key(seed, stream_id) + ctr);
  return (double)(h >> 11) * 0x1.0p-53;
}

namespace {

template <typename T>
__global__ void gaussian_kernel(T* __restrict__ out, int64_t n, int R, int64_t row0, uint64_t key,
                                double scale) {
  const int64_t total = n * R;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / R;
    const int q = static_cast<int>(i - r * R);
    const uint64_t ctr = (uint64_t)(row0 + r) * (uint64_t)R + (uint64_t)q;
    const uint64_t h1 = splitmix64_hd(key + 2ULL * ctr);
    const uint64_t h2 = splitmix64_hd(key + 2ULL * ctr + 1ULL);
    const double u1 = ((double)(h1 >> 11) + 1.0) * 0x1.0p-53;
    const double u2 = (double)(h2 >> 11) * 0x1.0p-53;
    const double z = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
    out[i] = static_cast<T>(z * scale);
  }
}

}  // namespace

template <typename T>
int random_signals(int64_t n, int R, int64_t row0, uint64_t seed, int stream_id, double variance,
                   T* out, cudaStream_t s) {
  if (variance <= 0.0) variance = 1.0 / R;
  const int64_t total = n * R;
  const int grid = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
  gaussian_kernel<T><<<grid, 256, 0, s>>>(out, n, R, row0, stream_key(seed, stream_id), std::sqrt(variance));
  SC_CUDA_TRY(cudaGetLastError());
  return SC_OK;
}
template int random_signals<float>(int64_t, int, int64_t, uint64_t, int, double, float*, cudaStream_t);
template int random_signals<double>(int64_t, int, int64_t, uint64_t, int, double, double*, cudaStream_t);

// ---------------------------------------------------------------------------
// Lanczos (fp64) for the largest Ritz value of L
// ---------------------------------------------------------------------------
namespace {

constexpr int kDotBlocks = 296;

// w = L v - beta_j v_prev   (one thread-group of 4 lanes per row)
__global__ void lanczos_spmv(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                             const float* __restrict__ val, const double* __restrict__ strength,
                             int64_t n, const double* __restrict__ v, const double* __restrict__ vprev,
                             const double* __restrict__ beta_j, double* __restrict__ w) {
  const int lane = threadIdx.x & 3;
  const double bj = beta_j ? *beta_j : 0.0;
  for (int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 2; row < n;
       row += ((int64_t)gridDim.x * blockDim.x) >> 2) {
    const int64_t b = row_ptr[row], e = row_ptr[row + 1];
    double acc = 0.0;
    for (int64_t k = b + lane; k < e; k += 4) acc += (val ? (double)val[k] : 1.0) * v[col[k]];
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
    if (lane == 0) w[row] = strength[row] * v[row] - acc - (vprev ? bj * vprev[row] : 0.0);
  }
}

// partial dot products (fixed grid) then fixed-order final sum -> deterministic
__global__ void dot_partial(const double* __restrict__ a, const double* __restrict__ b, int64_t n,
                            double* __restrict__ part) {
  __shared__ double sh[256];
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s += a[i] * b[i];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

__global__ void dot_final(const double* __restrict__ part, int nb, double* __restrict__ out) {
  __shared__ double sh[256];
  double s = 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) s += part[i];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

// w -= alpha v
__global__ void axpy_neg(double* __restrict__ w, const double* __restrict__ v, const double* __restrict__ alpha,
                         int64_t n) {
  const double al = *alpha;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    w[i] -= al * v[i];
}

// vnext = w / sqrt(b2); beta = sqrt(b2)
__global__ void scale_inv_sqrt(double* __restrict__ out, const double* __restrict__ w,
                               const double* __restrict__ b2, double* __restrict__ beta, int64_t n) {
  const double bb = sqrt(*b2);
  if (blockIdx.x == 0 && threadIdx.x == 0 && beta) *beta = bb;
  const double inv = bb > 0.0 ? 1.0 / bb : 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = w[i] * inv;
}

int dot(const double* a, const double* b, int64_t n, double* part, double* out, cudaStream_t s) {
  dot_partial<<<kDotBlocks, 256, 0, s>>>(a, b, n, part);
  dot_final<<<1, 256, 0, s>>>(part, kDotBlocks, out);
  SC_CUDA_TRY(cudaGetLastError());
  return SC_OK;
}

}  // namespace

// building blocks of the row-partitioned Lanczos (sc_dist.cu)
namespace lz {
int spmv(const sc_graph* g, const double* v, const double* vprev, const double* beta_j, double* w, cudaStream_t s) {
  const float* val = g->unit_weights ? nullptr : g->values.as<float>();
  lanczos_spmv<<<g->num_sms * 8, 256, 0, s>>>(g->row_ptr.as<int64_t>(), g->col_idx.as<int32_t>(), val,
                                                g->strength64.as<double>(), g->n_rows, v, vprev, beta_j, w);
  SC_CUDA_TRY(cudaGetLastError());
  return SC_OK;
}
int dot_local(const double* a, const double* b, int64_t n, double* part, double* out, cudaStream_t s) {
  return dot(a, b, n, part, out, s);
}
int axpy_neg(double* w, const double* v, const double* alpha, int64_t n, cudaStream_t s) {
  ::sc::axpy_neg<<<148 * 8, 256, 0, s>>>(w, v, alpha, n);
  SC_CUDA_TRY(cudaGetLastError());
  return SC_OK;
}
int scale_inv_sqrt(double* out, const double* w, const double* b2, double* beta, int64_t n, cudaStream_t s) {
  ::sc::scale_inv_sqrt<<<148 * 8, 256, 0, s>>>(out, w, b2, beta, n);
  SC_CUDA_TRY(cudaGetLastError());
  return SC_OK;
}
double theta_from(const std::vector<double>& ha, const std::vector<double>& hb) {
  const int iters = static_cast<int>(ha.size());
  int m = iters;
  for (int j = 1; j < iters; ++j) {
    if (!(hb[j] > 1e-12 * (std::fabs(ha[j - 1]) + 1e-300))) { m = j; break; }
  }
  std::vector<double> a(ha.begin(), ha.begin() + m), b(hb.begin() + 1, hb.begin() + m);
  return tridiag_max_eig(a, b);
}
}  // namespace lz

int lanczos_lambda_max(sc_graph* g, int iters, uint64_t seed, double* theta, cudaStream_t s) {
  const int64_t n = g->n_rows;
  // workspace: 3 vectors + w + partials + scalars (alpha[iters], b2[iters+1], beta[iters+1])
  const size_t vec = (size_t)n;
  SC_TRY(g->ws_misc.ensure(sizeof(double) * (4 * vec + kDotBlocks + 3 * (size_t)(iters + 2))));
  double* base = g->ws_misc.as<double>();
  double* v = base;
  double* vprev = v + vec;
  double* w = vprev + vec;
  double* tmp = w + vec;
  double* part = tmp + vec;
  double* alpha = part + kDotBlocks;
  double* b2 = alpha + (iters + 2);
  double* beta = b2 + (iters + 2);
  const int grid = g->num_sms * 8;

  // v_0 = r / ||r||
  SC_TRY(random_signals<double>(n, 1, 0, seed, 0, 1.0, tmp, s));
  SC_TRY(dot(tmp, tmp, n, part, b2, s));
  scale_inv_sqrt<<<grid, 256, 0, s>>>(v, tmp, b2, nullptr, n);
  SC_CUDA_TRY(cudaMemsetAsync(beta, 0, sizeof(double), s));
  const float* val = g->unit_weights ? nullptr : g->values.as<float>();
  for (int j = 0; j < iters; ++j) {
    lanczos_spmv<<<grid, 256, 0, s>>>(g->row_ptr.as<int64_t>(), g->col_idx.as<int32_t>(), val,
                                      g->strength64.as<double>(), n, v, j ? vprev : nullptr,
                                      beta + j, w);
    SC_TRY(dot(w, v, n, part, alpha + j, s));
    axpy_neg<<<grid, 256, 0, s>>>(w, v, alpha + j, n);
    SC_TRY(dot(w, w, n, part, b2 + j + 1, s));
    // rotate: vprev <- v, v <- w / beta
    std::swap(vprev, v);
    scale_inv_sqrt<<<grid, 256, 0, s>>>(v, w, b2 + j + 1, beta + j + 1, n);
    SC_CUDA_TRY(cudaGetLastError());
  }
  std::vector<double> ha(iters), hb(iters + 1);
  SC_CUDA_TRY(cudaMemcpyAsync(ha.data(), alpha, sizeof(double) * iters, cudaMemcpyDeviceToHost, s));
  SC_CUDA_TRY(cudaMemcpyAsync(hb.data(), beta, sizeof(double) * (iters + 1), cudaMemcpyDeviceToHost, s));
  SC_CUDA_TRY(cudaStreamSynchronize(s));
  // truncate at a (near) invariant subspace
  int m = iters;
  for (int j = 1; j < iters; ++j) {
    if (!(hb[j] > 1e-12 * (std::fabs(ha[j - 1]) + 1e-300))) { m = j; break; }
  }
  std::vector<double> a(ha.begin(), ha.begin() + m), b(hb.begin() + 1, hb.begin() + m);
  *theta = tridiag_max_eig(a, b);
  return SC_OK;
}

}  // namespace sc
