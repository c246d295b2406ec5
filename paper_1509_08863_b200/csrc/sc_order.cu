// Filter-order selection m*(lambda_c/lambda_N; delta) (§2.4 "Note on the choice of m",
// Eq. (4) l.151-162; §4.1 step 3 l.312), reading R18.
//
// The normalised filter h_r(lambda) = 1[lambda <= r] on [0, 1] (r = lambda_c/lambda_N) depends on
// r only (l.157-159).  For each candidate order m the polynomial the filter applies,
// p_m(lambda) = sum_{j<=m} g_j^(m) c_j T_j(2 lambda - 1) (sc_cheby_coeffs with lambda_max = 1),
// is compared with h_r on the grid G = {i/(n-1)} U {i min(1, 2r)/(n-1)}, i < n, minus the
// transition band [r(1-theta), r(1+theta)]; m* is the smallest m with max_G |h_r - p_m| <= delta.
//
// Device layout: one block per (order m, slice of the grid).  The block first writes the m+1
// coefficients of order m to shared memory (Jackson factors depend on m), then each thread
// evaluates p_m at its grid points by Clenshaw's recurrence in fp64; the block's max error is
// folded into err[m] with an integer atomicMax on the bit pattern (exact for non-negative
// doubles, so the result does not depend on the block order).  Orders are tried in batches of
// increasing size until one meets delta.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "sc_internal.cuh"

namespace sc {
namespace {

constexpr int kOrderThreads = 256;
constexpr int kOrderPtsPerThread = 8;

__global__ void __launch_bounds__(kOrderThreads)
order_error_kernel(double ratio, double theta, int jackson, int n_grid, int m_lo,
                   unsigned long long* __restrict__ err_bits) {
  extern __shared__ double d[];                       // m+1 coefficients of this block's order
  __shared__ double red[kOrderThreads / 32];
  const int m = m_lo + blockIdx.y;
  // c_0 = 1 - theta_c/pi, c_j = -2 sin(j theta_c)/(pi j); Jackson g_j with M = m+1 terms
  const double a = fmin(1.0, fmax(-1.0, 2.0 * ratio - 1.0));
  const double tc = acos(a);
  const double M = m + 1.0;
  const double q = M_PI / (M + 1.0);
  const double cotq = cos(q) / sin(q);
  for (int j = threadIdx.x; j <= m; j += blockDim.x) {
    double c = (j == 0) ? 1.0 - tc / M_PI : -2.0 * sin(j * tc) / (M_PI * j);
    if (jackson) c *= ((M - j + 1.0) * cos(j * q) + sin(j * q) * cotq) / (M + 1.0);
    d[j] = c;
  }
  __syncthreads();
  const double lo = ratio * (1.0 - theta), hi = ratio * (1.0 + theta);
  const double fine = fmin(1.0, 2.0 * ratio);
  const int total = 2 * n_grid;                        // two uniform grids, concatenated
  double e = 0.0;
  const int base = (blockIdx.x * kOrderThreads) * kOrderPtsPerThread + threadIdx.x;
#pragma unroll 1
  for (int t = 0; t < kOrderPtsPerThread; ++t) {
    const int g = base + t * kOrderThreads;
    if (g >= total) break;
    const int i = g < n_grid ? g : g - n_grid;
    const double lam = (double)i / (double)(n_grid - 1) * (g < n_grid ? 1.0 : fine);
    if (lam >= lo && lam <= hi) continue;
    const double x = 2.0 * lam - 1.0;
    // Clenshaw: b_k = d_k + 2x b_{k+1} - b_{k+2};  p = d_0 + x b_1 - b_2
    double b1 = 0.0, b2 = 0.0;
    for (int k = m; k >= 1; --k) {
      const double b0 = d[k] + 2.0 * x * b1 - b2;
      b2 = b1;
      b1 = b0;
    }
    const double p = d[0] + x * b1 - b2;
    const double h = lam <= ratio ? 1.0 : 0.0;
    e = fmax(e, fabs(h - p));
  }
  for (int o = 16; o > 0; o >>= 1) e = fmax(e, __shfl_xor_sync(0xffffffffu, e, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = e;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = red[0];
    for (int w = 1; w < kOrderThreads / 32; ++w) b = fmax(b, red[w]);
    atomicMax(&err_bits[blockIdx.y], (unsigned long long)__double_as_longlong(b));
  }
}

}  // namespace

int filter_order(double ratio, double delta, bool jackson, double theta, int n_grid, int m_max, int* m_star,
                 double* err_out, cudaStream_t s) {
  const int pts_per_block = kOrderThreads * kOrderPtsPerThread;
  const int gx = (2 * n_grid + pts_per_block - 1) / pts_per_block;
  unsigned long long* dev = nullptr;
  SC_CUDA_TRY(cudaMallocAsync(&dev, sizeof(unsigned long long) * (size_t)m_max, s));
  std::vector<unsigned long long> host(m_max);
  int found = 0, m_lo = 1, batch = 32;
  double last_err = NAN;
  int rc = SC_OK;
  while (m_lo <= m_max && !found) {
    const int cnt = std::min(batch, m_max - m_lo + 1);
    const size_t smem = sizeof(double) * (size_t)(m_lo + cnt);
    cudaError_t e = cudaMemsetAsync(dev, 0, sizeof(unsigned long long) * cnt, s);
    if (e == cudaSuccess && smem > 48 * 1024)
      e = cudaFuncSetAttribute(order_error_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess) {
      order_error_kernel<<<dim3(gx, cnt), kOrderThreads, smem, s>>>(ratio, theta, jackson ? 1 : 0, n_grid, m_lo, dev);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(host.data(), dev, sizeof(unsigned long long) * cnt, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
      rc = fail(SC_ERR_CUDA, std::string("filter_order: ") + cudaGetErrorString(e));
      break;
    }
    for (int i = 0; i < cnt; ++i) {
      double v;
      std::memcpy(&v, &host[i], sizeof v);
      last_err = v;
      if (v <= delta) {
        found = m_lo + i;
        break;
      }
    }
    m_lo += cnt;
    batch *= 2;
  }
  cudaFreeAsync(dev, s);
  if (rc != SC_OK) return rc;
  *m_star = found;
  if (err_out) *err_out = last_err;
  return SC_OK;
}

}  // namespace sc
