// Features -> clusters: row normalisation, k-means++ seeding, Lloyd iterations,
// adjusted Rand index.
//
// PAPER.md §2.2 step 4 (lines 109-113), §4.1 step 6 (lines 323-328): k-means with
// the Euclidean distance on the feature rows; §5: replicates.
// Decision arithmetic is fixed so that the result does not depend on thread
// scheduling (reading R8):
//   * distances: fp64, explicit differences, summed in ascending q with
//     __dsub_rn/__dmul_rn/__dadd_rn (no FMA contraction); large problems screen the
//     candidates in fp32 first with a rigorous error bound and compute the exact fp64
//     distance of the proven winner (undecided points get the exact full scan);
//   * centroid sums: members grouped by cluster (counting sort), exact 128-bit
//     fixed-point accumulation of the fp32 features (x * 2^(100-E), E the exponent
//     bound of max|x|; integer sums are order independent), rounded once to fp64
//     (= the correctly rounded sum, as math.fsum), then divided by the count.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "sc_internal.cuh"

namespace sc {

// Max dynamic shared memory of a kernel, grow-only and never below the 48 KB default:
// concurrent k-means calls (the stability scan's workers) with different sizes must not lower
// it under another call's launch.
static int smem_attr_at_least(const void* kern, int bytes) {
  static std::mutex mu;
  static std::vector<std::pair<const void*, int>> cur;
  std::lock_guard<std::mutex> lock(mu);
  for (auto& e : cur)
    if (e.first == kern) {
      if (bytes > e.second) {
        SC_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
        e.second = bytes;
      }
      return SC_OK;
    }
  const int v = std::max(bytes, 48 * 1024);
  SC_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, v));
  cur.emplace_back(kern, v);
  return SC_OK;
}
namespace {

constexpr int kB = 256;

__global__ void normalize_rows_kernel(float* __restrict__ F, int64_t n, int d) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float* r = F + i * d;
    double s = 0.0;
    for (int q = 0; q < d; ++q) s += (double)r[q] * (double)r[q];
    const double nrm = sqrt(s);
    if (nrm > 0.0)
      for (int q = 0; q < d; ++q) r[q] = (float)((double)r[q] / nrm);
  }
}

__global__ void absmax_bits_kernel(const float* __restrict__ F, int64_t total, unsigned* out) {
  unsigned m = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x)
    m = max(m, __float_as_uint(fabsf(F[i])));
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// Stage the rows [p0, p0 + kSP) of F into shared memory as fp32 [kSP][ld] (padded: the
// threads of a warp then read their own rows conflict-free), a warp per row, every copy of
// the tile in flight at once and no register holding the data.  When d % 4 == 0 (and F is
// 16-byte aligned) rows are copied with 16-byte cp.async into ld = d + 4 and read back as
// float4 (a quarter-warp's 8 rows then hit 32 distinct banks); otherwise 4-byte copies into
// ld = d + 1.  (4-byte copies saturated L1 -- 95 % of its throughput, 4 ms per check on
// configs[4] features -- where the 16-byte ones move the same bytes in a quarter of the
// requests.)
constexpr int kSP = 128;   // points per block of the per-point kernels
__device__ __forceinline__ bool rows_v4(const float* F, int d) {
  return (d & 3) == 0 && (reinterpret_cast<uintptr_t>(F) & 15) == 0;
}
__device__ __forceinline__ int rows_ld(bool v4, int d) { return v4 ? d + 4 : d + 1; }
// copy row `src` (d floats) to `dst` with the calling warp
__device__ __forceinline__ void stage_row(const float* __restrict__ src, float* __restrict__ dst, int d, bool v4,
                                          int lane) {
  if (v4) {
    for (int v = lane; v < (d >> 2); v += 32) {
      const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(dst + 4 * v));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(src + 4 * v) : "memory");
    }
  } else {
    for (int q = lane; q < d; q += 32) {
      const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(dst + q));
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(src + q) : "memory");
    }
  }
}
__device__ __forceinline__ void stage_rows(const float* __restrict__ F, int64_t n, int d, int64_t p0,
                                           float* __restrict__ sx, bool v4) {
  const int rows = (int)min((int64_t)kSP, n - p0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int ld = rows_ld(v4, d);
  for (int r = warp; r < rows; r += nw) stage_row(F + (p0 + r) * d, sx + r * ld, d, v4, lane);
  asm volatile("cp.async.wait_all;" ::: "memory");
}
// exact squared distance of a staged row to centre c (R8: explicit sub/mul/add in ascending q)
__device__ __forceinline__ double row_dist(const float* __restrict__ x, const double* __restrict__ c, int d, bool v4) {
  double acc = 0.0;
  if (v4) {
    for (int q = 0; q < d; q += 4) {
      const float4 v = *reinterpret_cast<const float4*>(x + q);
      const float xs[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double diff = __dsub_rn((double)xs[u], c[q + u]);
        acc = __dadd_rn(acc, __dmul_rn(diff, diff));
      }
    }
  } else {
    for (int q = 0; q < d; ++q) {
      const double diff = __dsub_rn((double)x[q], c[q]);
      acc = __dadd_rn(acc, __dmul_rn(diff, diff));
    }
  }
  return acc;
}

// d2[i] = (first ? dist : min(d2[i], dist)) to centre c (device fp64 row)
__global__ void __launch_bounds__(kSP) d2_update_kernel(const float* __restrict__ F, int64_t n, int d,
                                                        const double* __restrict__ c, double* __restrict__ d2,
                                                        int first, int32_t* __restrict__ near) {
  extern __shared__ unsigned char smd[];
  double* sc_ = reinterpret_cast<double*>(smd);
  float* sx = reinterpret_cast<float*>(sc_ + d);
  for (int q = threadIdx.x; q < d; q += blockDim.x) sc_[q] = c[q];
  const int64_t p0 = (int64_t)blockIdx.x * kSP;
  const bool v4 = rows_v4(F, d);
  stage_rows(F, n, d, p0, sx, v4);
  __syncthreads();
  const int64_t i = p0 + threadIdx.x;
  if (i < n) {
    const double acc = row_dist(sx + threadIdx.x * rows_ld(v4, d), sc_, d, v4);
    d2[i] = first ? acc : fmin(d2[i], acc);
    if (first && near) near[i] = 0;
  }
}

// D^2 update for seed t >= 1 with the triangle inequality: if the point's distance r to its
// nearest seed j satisfies r (1 + 1e-9) <= half_gap[j] (= ||c_t - c_j|| / 2, rounded down),
// then ||x - c_t|| >= ||c_t - c_j|| - r >= r (1 + 1e-9) and the computed new D^2 exceeds the
// computed d2 (both carry < 1e-13 relative rounding): min(d2, new) = d2 exactly as in the
// full computation, so the row is not read.  Other points: the exact R8 distance.
// One block per kSP consecutive points: the skip test first (coalesced d2 / near reads), the
// surviving points compacted, only their rows staged into shared memory (a warp per row,
// lanes along the row: coalesced), then each survivor's distance summed by its own thread in
// ascending q (R8).  (A thread-per-point version read every row with a stride of d floats
// between lanes: 3.4 ms per seed on configs[4], 3x the full coalesced update.)
__global__ void __launch_bounds__(kSP) d2_update_skip_kernel(const float* __restrict__ F, int64_t n, int d,
                                                             const double* __restrict__ c, int t,
                                                             const double* __restrict__ half_gap,
                                                             double* __restrict__ d2, int32_t* __restrict__ near) {
  extern __shared__ unsigned char smk[];
  double* sct = reinterpret_cast<double*>(smk);
  float* sx = reinterpret_cast<float*>(sct + d);   // [kSP][d + 1]
  __shared__ int s_cnt;
  __shared__ int s_rows[kSP];
  for (int q = threadIdx.x; q < d; q += blockDim.x) sct[q] = c[q];
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  const int64_t p0 = (int64_t)blockIdx.x * kSP;
  const int64_t i = p0 + threadIdx.x;
  double cur = 0.0;
  if (i < n) {
    cur = d2[i];
    if (!(sqrt(cur) * (1.0 + 1e-9) <= half_gap[near[i]])) s_rows[atomicAdd(&s_cnt, 1)] = threadIdx.x;
  }
  __syncthreads();
  const int cnt = s_cnt;
  if (cnt == 0) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const bool v4 = rows_v4(F, d);
  const int ld = rows_ld(v4, d);
  for (int r = warp; r < cnt; r += nw) stage_row(F + (p0 + s_rows[r]) * d, sx + r * ld, d, v4, lane);
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  if ((int)threadIdx.x < cnt) {
    const int lr = s_rows[threadIdx.x];
    const int64_t gi = p0 + lr;
    const double acc = row_dist(sx + threadIdx.x * ld, sct, d, v4);
    if (acc < d2[gi]) {
      d2[gi] = acc;
      near[gi] = t;
    }
  }
}

// per-block sums of d2 over contiguous ranges [b*chunk, (b+1)*chunk)
__global__ void range_sums_kernel(const double* __restrict__ v, int64_t n, int64_t chunk, double* __restrict__ out) {
  __shared__ double sh[kB];
  const int64_t b0 = blockIdx.x * chunk, b1 = min(n, b0 + chunk);
  double s = 0.0;
  for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) s += v[i];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = kB / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = sh[0];
}

// Whole k-means++ draw on the device (no host round trip), one 1024-thread block: the G
// block sums are prefixed (fixed-order block scan), the block holding u * total is found,
// its range is split into 1024 contiguous slices whose sums are prefixed the same way, and
// the slice crossing the target is scanned sequentially for the first i with
// prefix_i > u * total (R13: a fixed summation order of the GPU's own).  The
// chosen row is copied into centroid slot `c_out`.  total <= 0 (all points coincide with
// centres): uniform draw floor(u n).
constexpr int kSel = 1024;
// inclusive block scan in a fixed order (warp shuffle scans, then the warp totals); every
// thread's inclusive value lands in s_inc[threadIdx.x]
__device__ __forceinline__ void block_inclusive_scan(double v, double* s_w, double* s_inc) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_w[warp] = x;
  __syncthreads();
  if (warp == 0) {
    double t = s_w[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    s_w[32 + lane] = t;
  }
  __syncthreads();
  s_inc[threadIdx.x] = (warp ? s_w[32 + warp - 1] : 0.0) + x;
  __syncthreads();
}

__device__ __forceinline__ void seed_select_dev(const double* __restrict__ bsum, int G,
                                                const double* __restrict__ v, int64_t n, int64_t chunk,
                                                double u, const float* __restrict__ F, int d,
                                                double* __restrict__ c_out, int tseed,
                                                double* __restrict__ half_gap) {
  __shared__ double s_w[64];
  __shared__ double s_inc[kSel];
  __shared__ int s_first;
  __shared__ long long s_idx, s_last;
  const int t = threadIdx.x;
  // 1. prefix of the G <= kSel block sums; the chosen block is the first whose inclusive
  // prefix exceeds u * total (atomicMin: unique even if rounding made the prefix non-monotone)
  block_inclusive_scan(t < G ? bsum[t] : 0.0, s_w, s_inc);
  const double total = s_inc[kSel - 1];
  if (t == 0) { s_first = INT_MAX; s_last = -1; }
  __syncthreads();
  if (!(total > 0.0)) {
    if (t == 0) {
      const long long idx = (long long)floor(u * (double)n);
      s_idx = idx < n - 1 ? idx : n - 1;
    }
    __syncthreads();
  } else {
    const double target = u * total;
    if (t < G && s_inc[t] > target) atomicMin(&s_first, t);
    __syncthreads();
    const int blk = s_first == INT_MAX ? G - 1 : s_first;
    const double start = blk ? s_inc[blk - 1] : 0.0;
    __syncthreads();
    // 2. kSel contiguous slices of the chosen block, prefixed the same way
    const int64_t b0 = (int64_t)blk * chunk, b1 = min(n, b0 + chunk);
    const int64_t len = b1 - b0 > 0 ? b1 - b0 : 0;
    const int64_t per = (len + kSel - 1) / kSel;
    const int64_t s0 = min(b1, b0 + t * per), s1 = min(b1, s0 + per);
    double sum = 0.0;
    long long last_pos = -1;
    for (int64_t i = s0; i < s1; ++i) {
      const double vi = v[i];
      sum += vi;
      if (vi > 0.0) last_pos = i;
    }
    if (last_pos >= 0) atomicMax(&s_last, last_pos);
    if (t == 0) s_first = INT_MAX;
    block_inclusive_scan(sum, s_w, s_inc);
    if (s1 > s0 && start + s_inc[t] > target) atomicMin(&s_first, t);
    __syncthreads();
    if (s_first == INT_MAX) {
      if (t == 0) s_idx = s_last >= 0 ? s_last : b1 - 1;
    } else if (t == s_first) {
      double acc = start + (t ? s_inc[t - 1] : 0.0);
      long long pick = s1 - 1;
      for (int64_t i = s0; i < s1; ++i) {
        acc += v[i];
        if (acc > target) { pick = i; break; }
      }
      s_idx = pick;
    }
    __syncthreads();
  }
  const int64_t idx = s_idx;
  for (int q = t; q < d; q += blockDim.x) c_out[q] = (double)F[idx * d + q];
  if (half_gap) {
    // half distances from the new seed (c_out = C[tseed]) to the earlier seeds C[0..tseed-1],
    // rounded down (d2_update_skip_kernel's triangle test)
    __syncthreads();
    for (int j = t; j < tseed; j += blockDim.x) {
      double s2 = 0.0;
      for (int q = 0; q < d; ++q) {
        const double df = c_out[q] - c_out[(int64_t)(j - tseed) * d + q];
        s2 += df * df;
      }
      half_gap[j] = 0.5 * sqrt(s2) * (1.0 - 1e-9);
    }
  }
}

__global__ void __launch_bounds__(kSel) seed_select_kernel(const double* __restrict__ bsum, int G,
                                                           const double* __restrict__ v, int64_t n, int64_t chunk,
                                                           double u, const float* __restrict__ F, int d,
                                                           double* __restrict__ c_out, int tseed,
                                                           double* __restrict__ half_gap) {
  seed_select_dev(bsum, G, v, n, chunk, u, F, d, c_out, tseed, half_gap);
}

// ---- k-means++ of several restarts at once (kmeans_run with parallel restarts): the draws of
// all restarts advance together, one launch per step for all of them, and a feature row is read
// once per draw index for every restart that needs it (the per-restart path reads it once per
// restart).  Each restart's arithmetic is exactly the per-restart path's -- the same row_dist,
// range sums, selection and skip test -- so the seeds are identical (restart r's arrays at
// offset r of the batch).
__global__ void __launch_bounds__(kSel) seed_select_batch_kernel(const double* __restrict__ bsum_all, int G,
                                                                 const double* __restrict__ v_all, int64_t n,
                                                                 int64_t chunk, const double* __restrict__ u_all,
                                                                 int ustride, const float* __restrict__ F, int d,
                                                                 double* __restrict__ C_all, int64_t cstride, int tseed,
                                                                 double* __restrict__ gap_all, int gstride) {
  const int r = blockIdx.x;
  seed_select_dev(bsum_all + (size_t)r * G, G, v_all + (size_t)r * n, n, chunk, u_all[(size_t)r * ustride + tseed], F,
                  d, C_all + (size_t)r * cstride + (size_t)tseed * d, tseed, gap_all + (size_t)r * gstride);
}

// d2 of every restart to its first seed (d2_update_kernel with first = 1, per restart)
__global__ void __launch_bounds__(kSP) d2_first_batch_kernel(const float* __restrict__ F, int64_t n, int d,
                                                             const double* __restrict__ C_all, int64_t cstride, int nr,
                                                             double* __restrict__ d2_all, int32_t* __restrict__ near_all) {
  extern __shared__ unsigned char smb[];
  double* sc_ = reinterpret_cast<double*>(smb);        // [nr][d]
  float* sx = reinterpret_cast<float*>(sc_ + (size_t)nr * d);
  for (int j = threadIdx.x; j < nr * d; j += blockDim.x) sc_[j] = C_all[(size_t)(j / d) * cstride + j % d];
  const int64_t p0 = (int64_t)blockIdx.x * kSP;
  const bool v4 = rows_v4(F, d);
  stage_rows(F, n, d, p0, sx, v4);
  __syncthreads();
  const int64_t i = p0 + threadIdx.x;
  if (i < n) {
    const float* x = sx + threadIdx.x * rows_ld(v4, d);
    for (int r = 0; r < nr; ++r) {
      d2_all[(size_t)r * n + i] = row_dist(x, sc_ + (size_t)r * d, d, v4);
      near_all[(size_t)r * n + i] = 0;
    }
  }
}

// seed t of every restart: d2_update_skip_kernel's test per (point, restart); a row is staged
// once if any restart needs it, then each needing restart's exact distance (R8) is taken
__global__ void __launch_bounds__(kSP) d2_skip_batch_kernel(const float* __restrict__ F, int64_t n, int d,
                                                            const double* __restrict__ C_all, int64_t cstride, int t,
                                                            int nr, const double* __restrict__ gap_all, int gstride,
                                                            double* __restrict__ d2_all,
                                                            int32_t* __restrict__ near_all) {
  extern __shared__ unsigned char smk2[];
  double* sct = reinterpret_cast<double*>(smk2);   // [nr][d]: seed t of every restart
  float* sx = reinterpret_cast<float*>(sct + (size_t)nr * d);
  __shared__ int s_cnt;
  __shared__ int s_rows[kSP];
  __shared__ unsigned s_mask[kSP];
  for (int j = threadIdx.x; j < nr * d; j += blockDim.x)
    sct[j] = C_all[(size_t)(j / d) * cstride + (size_t)t * d + j % d];
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  const int64_t p0 = (int64_t)blockIdx.x * kSP;
  const int64_t i = p0 + threadIdx.x;
  unsigned mask = 0;
  if (i < n) {
    for (int r = 0; r < nr; ++r) {
      const double cur = d2_all[(size_t)r * n + i];
      if (!(sqrt(cur) * (1.0 + 1e-9) <= gap_all[(size_t)r * gstride + near_all[(size_t)r * n + i]])) mask |= 1u << r;
    }
    if (mask) {
      const int slot = atomicAdd(&s_cnt, 1);
      s_rows[slot] = threadIdx.x;
      s_mask[slot] = mask;
    }
  }
  __syncthreads();
  const int cnt = s_cnt;
  if (cnt == 0) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const bool v4 = rows_v4(F, d);
  const int ld = rows_ld(v4, d);
  for (int q = warp; q < cnt; q += nw) stage_row(F + (p0 + s_rows[q]) * d, sx + q * ld, d, v4, lane);
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  if ((int)threadIdx.x < cnt) {
    const int64_t gi = p0 + s_rows[threadIdx.x];
    unsigned m = s_mask[threadIdx.x];
    const float* x = sx + threadIdx.x * ld;
    while (m) {
      const int r = __ffs(m) - 1;
      m &= m - 1;
      const double acc = row_dist(x, sct + (size_t)r * d, d, v4);
      if (acc < d2_all[(size_t)r * n + gi]) {
        d2_all[(size_t)r * n + gi] = acc;
        near_all[(size_t)r * n + gi] = t;
      }
    }
  }
}

// per-block sums of every restart's d2 (range_sums_kernel per restart: blockIdx.y)
__global__ void range_sums_batch_kernel(const double* __restrict__ v_all, int64_t n, int64_t chunk, int G,
                                        double* __restrict__ out_all) {
  __shared__ double sh[kB];
  const double* v = v_all + (size_t)blockIdx.y * n;
  const int64_t b0 = blockIdx.x * chunk, b1 = min(n, b0 + chunk);
  double s = 0.0;
  for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) s += v[i];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = kB / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out_all[(size_t)blockIdx.y * G + blockIdx.x] = sh[0];
}

// ---- distributed k-means++ (kmeans_run_dist): the points are the ranks' rows in rank-major
// order.  Each rank sums its D^2 in the same fixed order as seed_select_kernel (block sums,
// then a block scan of them); the per-rank totals are summed over the ranks (S_all, every
// entry but this rank's zero before the all-reduce), the draw's owner is the first rank whose
// cumulative total exceeds u * total, and it selects its row exactly as seed_select_kernel does
// with its local target; the other ranks write zeros and the row reaches every rank through
// the sum all-reduce (x + 0 = x).  DESIGN.md R13: the global prefix is summed per rank here.
__global__ void __launch_bounds__(kSel) local_total_kernel(const double* __restrict__ bsum, int G, int rank,
                                                           double* __restrict__ s_all) {
  __shared__ double s_w[64];
  __shared__ double s_inc[kSel];
  block_inclusive_scan(threadIdx.x < G ? bsum[threadIdx.x] : 0.0, s_w, s_inc);
  if (threadIdx.x == 0) s_all[rank] = s_inc[kSel - 1];
}

struct DistDraw {
  int rank, world;
  int64_t row_off, n_global;
};

__global__ void __launch_bounds__(kSel) seed_select_dist_kernel(const double* __restrict__ bsum, int G,
                                                                const double* __restrict__ v, int64_t n,
                                                                int64_t chunk, double u,
                                                                const double* __restrict__ s_all, DistDraw dd,
                                                                const float* __restrict__ F, int d,
                                                                double* __restrict__ c_out) {
  __shared__ double s_w[64];
  __shared__ double s_inc[kSel];
  __shared__ int s_first;
  __shared__ long long s_idx, s_last;
  const int t = threadIdx.x;
  double total = 0.0, pre = 0.0;
  int owner = -1;
  for (int q = 0; q < dd.world; ++q) total += s_all[q];
  long long gidx = -1;   // uniform draw (all D^2 zero): global index
  double target = 0.0;
  if (!(total > 0.0)) {
    const long long idx = (long long)floor(u * (double)dd.n_global);
    gidx = idx < dd.n_global - 1 ? idx : dd.n_global - 1;
    owner = (gidx >= dd.row_off && gidx < dd.row_off + n) ? dd.rank : -1;
  } else {
    target = u * total;
    double cum = 0.0;
    int last_pos = -1;
    for (int q = 0; q < dd.world; ++q) {
      if (s_all[q] > 0.0) last_pos = q;
      if (owner < 0 && cum + s_all[q] > target) { owner = q; pre = cum; }
      cum += s_all[q];
    }
    if (owner < 0) {   // rounding: the last rank holding positive D^2 takes the draw
      owner = last_pos;
      pre = 0.0;
      for (int q = 0; q < last_pos; ++q) pre += s_all[q];
    }
  }
  if (owner != dd.rank) {
    for (int q = t; q < d; q += blockDim.x) c_out[q] = 0.0;
    return;
  }
  if (gidx >= 0) {
    const int64_t idx = gidx - dd.row_off;
    for (int q = t; q < d; q += blockDim.x) c_out[q] = (double)F[idx * d + q];
    return;
  }
  // this rank owns the draw: local target, then exactly seed_select_kernel's two-level search
  const double ltarget = target - pre;
  block_inclusive_scan(t < G ? bsum[t] : 0.0, s_w, s_inc);
  if (t == 0) { s_first = INT_MAX; s_last = -1; }
  __syncthreads();
  if (t < G && s_inc[t] > ltarget) atomicMin(&s_first, t);
  __syncthreads();
  const int blk = s_first == INT_MAX ? G - 1 : s_first;
  const double start = blk ? s_inc[blk - 1] : 0.0;
  __syncthreads();
  const int64_t b0 = (int64_t)blk * chunk, b1 = min(n, b0 + chunk);
  const int64_t len = b1 - b0 > 0 ? b1 - b0 : 0;
  const int64_t per = (len + kSel - 1) / kSel;
  const int64_t s0 = min(b1, b0 + t * per), s1 = min(b1, s0 + per);
  double sum = 0.0;
  long long last_pos = -1;
  for (int64_t i = s0; i < s1; ++i) {
    const double vi = v[i];
    sum += vi;
    if (vi > 0.0) last_pos = i;
  }
  if (last_pos >= 0) atomicMax(&s_last, last_pos);
  if (t == 0) s_first = INT_MAX;
  block_inclusive_scan(sum, s_w, s_inc);
  if (s1 > s0 && start + s_inc[t] > ltarget) atomicMin(&s_first, t);
  __syncthreads();
  if (s_first == INT_MAX) {
    if (t == 0) s_idx = s_last >= 0 ? s_last : b1 - 1;
  } else if (t == s_first) {
    double acc = start + (t ? s_inc[t - 1] : 0.0);
    long long pick = s1 - 1;
    for (int64_t i = s0; i < s1; ++i) {
      acc += v[i];
      if (acc > ltarget) { pick = i; break; }
    }
    s_idx = pick;
  }
  __syncthreads();
  const int64_t idx = s_idx;
  for (int q = t; q < d; q += blockDim.x) c_out[q] = (double)F[idx * d + q];
}

// half distances from seed tseed to the earlier seeds (as seed_select_kernel computes them)
__global__ void half_gap_kernel(const double* __restrict__ C, int d, int tseed, double* __restrict__ half_gap) {
  const double* c_out = C + (int64_t)tseed * d;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < tseed; j += gridDim.x * blockDim.x) {
    double s2 = 0.0;
    for (int q = 0; q < d; ++q) {
      const double df = c_out[q] - C[(int64_t)j * d + q];
      s2 += df * df;
    }
    half_gap[j] = 0.5 * sqrt(s2) * (1.0 - 1e-9);
  }
}

__global__ void row_or_zero_kernel(const float* __restrict__ F, int64_t idx_local, int d, double* __restrict__ c) {
  for (int q = threadIdx.x; q < d; q += blockDim.x) c[q] = idx_local >= 0 ? (double)F[idx_local * d + q] : 0.0;
}

__global__ void row_to_centroid_kernel(const float* __restrict__ F, int64_t idx, int d, double* __restrict__ c) {
  for (int q = threadIdx.x; q < d; q += blockDim.x) c[q] = (double)F[idx * d + q];
}

// exact fixed-point image of an fp32 value: x * 2^shift as a signed 128-bit integer
__device__ __forceinline__ __int128 to_fixed(float xf, int shift) {
  const unsigned u = __float_as_uint(xf);
  const int ef = (u >> 23) & 0xff;
  unsigned long long m = u & 0x7fffffu;
  int e;
  if (ef == 0) e = -149;
  else { m |= 0x800000u; e = ef - 150; }
  if (m == 0) return 0;
  const int s = e + shift;
  __int128 v;
  if (s >= 0) v = (__int128)m << s;
  else if (s > -40) v = (__int128)((m + (1ull << (-s - 1))) >> (-s));
  else v = 0;
  return (u >> 31) ? -v : v;
}

// correctly rounded double of S * 2^-shift, S a signed 128-bit integer
__device__ double fixed_to_double(__int128 S, int shift) {
  if (S == 0) return 0.0;
  const bool neg = S < 0;
  unsigned __int128 u = neg ? (unsigned __int128)(-S) : (unsigned __int128)S;
  const unsigned long long hi = (unsigned long long)(u >> 64), lo = (unsigned long long)u;
  const int bits = hi ? 128 - __clzll(hi) : 64 - __clzll(lo);
  double r;
  if (bits <= 53) {
    r = (double)lo;
  } else {
    const int s = bits - 53;
    unsigned __int128 m = u >> s;
    const unsigned __int128 rem = u & (((unsigned __int128)1 << s) - 1);
    const unsigned __int128 half = (unsigned __int128)1 << (s - 1);
    if (rem > half || (rem == half && (m & 1))) m += 1;
    r = ldexp((double)(unsigned long long)m, s);
  }
  r = ldexp(r, -shift);
  return neg ? -r : r;
}

__global__ void contingency_kernel(const int32_t* __restrict__ a, const int32_t* __restrict__ b, int64_t n,
                                   int ka, int kb, unsigned long long* __restrict__ t) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&t[(int64_t)a[i] * kb + b[i]], 1ull);
}

__global__ void minmax_kernel(const int32_t* __restrict__ a, int64_t n, int* out /*[2]: min,max*/) {
  int mn = INT_MAX, mx = INT_MIN;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    mn = min(mn, a[i]);
    mx = max(mx, a[i]);
  }
  for (int o = 16; o > 0; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if ((threadIdx.x & 31) == 0) { atomicMin(out, mn); atomicMax(out + 1, mx); }
}


// ---------------------------------------------------------------------------
// Lloyd assignment, register-tiled like a GEMM: a block of 256 threads computes the
// distances of 64 points to centroid tiles of 64; thread (ty, tx) owns 4 points x 4
// centroids (16 fp64 accumulators).  Points and centroids are staged as fp64 [d][64]
// in shared memory.  Distance = sum_q (x_q - c_q)^2 in ascending q with
// __dsub_rn/__dmul_rn/__dadd_rn (R8); each thread keeps the first minimum over
// its centroids, the 16 threads of a point row reduce (dist, index) lexicographically,
// so the result is the lowest index among equal minima, as np.argmin.
// ---------------------------------------------------------------------------
constexpr int kAT = 64;   // points per block and centroids per tile

// Full scan of the points in `list` (or all points when list == nullptr): exact argmin
// (first minimum) and the second-smallest distance, which becomes the point's lower bound
// lo_i = sqrt(second) for the pruning test of the next iterations (check_kernel).
// NC centroids per thread (tx, tx+16, ...): centroid tiles of 16 NC columns, so small k is not
// padded to 64 (k = 10 computes 16 columns, k = 20 or 30 computes 32)
template <int NC>
__global__ void __launch_bounds__(256) assign3_kernel(const float* __restrict__ F, int64_t n, int d,
                                                      const double* __restrict__ C, int k,
                                                      const int32_t* __restrict__ list, const int* __restrict__ list_len,
                                                      int32_t* __restrict__ lab, double* __restrict__ dmin,
                                                      double* __restrict__ lo) {
  extern __shared__ double sm3[];
  double* sX = sm3;                        // [d][kAT]
  double* sC = sm3 + (size_t)d * kAT;      // [d][kAT]
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int64_t m = list ? (int64_t)*list_len : n;
  // grid-stride over 64-point tiles (list mode is launched with a bounded grid: the list
  // length is only known on the device)
  for (int64_t p0 = (int64_t)blockIdx.x * kAT; p0 < m; p0 += (int64_t)gridDim.x * kAT) {
  __syncthreads();   // previous tile's shared-memory reads done
  // staging with 8 independent loads in flight per thread
  for (int e0 = tid; e0 < kAT * d; e0 += 256 * 8) {
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * 256;
      v[u] = 0.f;
      if (e < kAT * d) {
        const int row = e / d, q = e - row * d;
        const int64_t pi = p0 + row;
        const int64_t gi = pi < m ? (list ? (int64_t)list[pi] : pi) : -1;
        if (gi >= 0) v[u] = __ldg(F + gi * d + q);
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * 256;
      if (e < kAT * d) {
        const int row = e / d, q = e - row * d;
        sX[(size_t)q * kAT + row] = (double)v[u];
      }
    }
  }
  double best[4], second[4];
  int bidx[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) { best[i] = INFINITY; second[i] = INFINITY; bidx[i] = -1; }
  constexpr int TW = 16 * NC;   // centroids per tile
  for (int c0 = 0; c0 < k; c0 += TW) {
    const int kt = min(TW, k - c0);
    __syncthreads();
    for (int e0 = tid; e0 < TW * d; e0 += 256 * 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * 256;
        v[u] = 0.0;
        if (e < TW * d) {
          const int cc = e / d, q = e - cc * d;
          if (cc < kt) v[u] = __ldg(C + (size_t)(c0 + cc) * d + q);
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * 256;
        if (e < TW * d) {
          const int cc = e / d, q = e - cc * d;
          sC[(size_t)q * kAT + cc] = v[u];
        }
      }
    }
    __syncthreads();
    double acc[4][NC];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < NC; ++j) acc[i][j] = 0.0;
#pragma unroll 2
    for (int q = 0; q < d; ++q) {
      const double2 xa = *reinterpret_cast<const double2*>(sX + (size_t)q * kAT + ty * 4);
      const double2 xb = *reinterpret_cast<const double2*>(sX + (size_t)q * kAT + ty * 4 + 2);
      // thread tx owns centroids tx, tx+16, ... of the tile: the 16 lanes of a row read 16
      // consecutive doubles per load (one wavefront, no bank conflicts)
      const double* cq = sC + (size_t)q * kAT + tx;
      const double xv[4] = {xa.x, xa.y, xb.x, xb.y};
      double cv[NC];
#pragma unroll
      for (int j = 0; j < NC; ++j) cv[j] = cq[16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < NC; ++j) {
          const double diff = __dsub_rn(xv[i], cv[j]);
          acc[i][j] = __dadd_rn(acc[i][j], __dmul_rn(diff, diff));
        }
    }
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      const int cidx = tx + 16 * j;
      if (cidx < kt) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const double v = acc[i][j];
          if (v < best[i]) { second[i] = best[i]; best[i] = v; bidx[i] = c0 + cidx; }
          else if (v < second[i]) second[i] = v;
        }
      }
    }
  }
  // (dist, index) lexicographic min over the 16 threads of each point row, second best merged
#pragma unroll
  for (int i = 0; i < 4; ++i) {
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best[i], o);
      const double os = __shfl_xor_sync(0xffffffffu, second[i], o);
      const int oi = __shfl_xor_sync(0xffffffffu, bidx[i], o);
      const bool take = (oi >= 0) && (bidx[i] < 0 || ob < best[i] || (ob == best[i] && oi < bidx[i]));
      const double loser = take ? best[i] : ob;
      second[i] = fmin(fmin(second[i], os), loser);
      if (take) { best[i] = ob; bidx[i] = oi; }
    }
  }
  // thread tx < 4 of row ty handles point ty*4 + tx
  const int i = tx & 3;
  double bv = best[0], sv = second[0];
  int bl = bidx[0];
#pragma unroll
  for (int ii = 1; ii < 4; ++ii) if (ii == i) { bv = best[ii]; sv = second[ii]; bl = bidx[ii]; }
  const int64_t pi = p0 + ty * 4 + i;
  if (tx < 4 && pi < m) {
    const int64_t gi = list ? (int64_t)list[pi] : pi;
    if (bl < 0) bl = 0;   // all distances NaN/inf: deterministic fallback
    lab[gi] = bl;
    dmin[gi] = bv;
    lo[gi] = sqrt(sv);
  }
  }
}

// Exact scan of a short list of points (the screens' ambiguous points): one warp per point,
// lane l owns centroids l, l + 32, l + 64, l + 96 (four independent fp64 chains), the
// centroids transposed in shared memory ([d][k], loaded once per block), the point's row
// broadcast from a per-warp shared-memory copy.  Same arithmetic and decisions as
// assign3_kernel: sum_q (x_q - c_q)^2 in ascending q with __dsub_rn/__dmul_rn/__dadd_rn, first
// minimum (lowest index on ties), second-smallest distance -> lo (R8).  Used when
// k <= 128 and k d doubles fit in shared memory; the tile kernel above serves the rest.
constexpr int kAmbK = 128;   // centroids per point pass: 4 per lane
__global__ void __launch_bounds__(256) amb_scan_kernel(const float* __restrict__ F, int d,
                                                       const double* __restrict__ C, int k,
                                                       const int32_t* __restrict__ list,
                                                       const int* __restrict__ list_len,
                                                       int32_t* __restrict__ lab, double* __restrict__ dmin,
                                                       double* __restrict__ lo) {
  extern __shared__ double smA[];
  double* sCt = smA;                          // [d][k]
  double* sXw = smA + (size_t)d * k;          // [8 warps][d]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m = *list_len;
  if ((int64_t)blockIdx.x * 8 >= m) return;
  for (int e = tid; e < k * d; e += 256) {
    const int j = e / d, q = e - j * d;
    sCt[(size_t)q * k + j] = C[e];
  }
  __syncthreads();
  double* xw = sXw + (size_t)warp * d;
  for (int pi = blockIdx.x * 8 + warp; pi < m; pi += gridDim.x * 8) {
    const int64_t gi = list[pi];
    for (int q = lane; q < d; q += 32) xw[q] = (double)__ldg(F + gi * d + q);
    __syncwarp();
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    const bool v0 = lane < k, v1 = lane + 32 < k, v2 = lane + 64 < k, v3 = lane + 96 < k;
    const double* c0 = sCt + (v0 ? lane : 0);
    const double* c1 = sCt + (v1 ? lane + 32 : 0);
    const double* c2 = sCt + (v2 ? lane + 64 : 0);
    const double* c3 = sCt + (v3 ? lane + 96 : 0);
#pragma unroll 4
    for (int q = 0; q < d; ++q) {
      const double x = xw[q];
      const size_t o = (size_t)q * k;
      const double d0 = __dsub_rn(x, c0[o]), d1 = __dsub_rn(x, c1[o]);
      const double d2 = __dsub_rn(x, c2[o]), d3 = __dsub_rn(x, c3[o]);
      acc[0] = __dadd_rn(acc[0], __dmul_rn(d0, d0));
      acc[1] = __dadd_rn(acc[1], __dmul_rn(d1, d1));
      acc[2] = __dadd_rn(acc[2], __dmul_rn(d2, d2));
      acc[3] = __dadd_rn(acc[3], __dmul_rn(d3, d3));
    }
    __syncwarp();   // xw reused by the warp's next point
    // this lane's centroids in ascending index, then the (dist, index) lexicographic min over
    // the warp with the second-smallest distance merged (as assign3_kernel)
    double best = INFINITY, second = INFINITY;
    int bidx = -1;
    const bool valid[4] = {v0, v1, v2, v3};
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      if (!valid[t]) continue;
      const double v = acc[t];
      if (v < best) { second = best; best = v; bidx = lane + 32 * t; }
      else if (v < second) second = v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const double os = __shfl_xor_sync(0xffffffffu, second, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
      const bool take = (oi >= 0) && (bidx < 0 || ob < best || (ob == best && oi < bidx));
      const double loser = take ? best : ob;
      second = fmin(fmin(second, os), loser);
      if (take) { best = ob; bidx = oi; }
    }
    if (lane == 0) {
      lab[gi] = bidx < 0 ? 0 : bidx;   // all distances NaN/inf: deterministic fallback
      dmin[gi] = best;
      lo[gi] = sqrt(second);
    }
  }
}

// ---------------------------------------------------------------------------
// Screened assignment: an fp32 pass finds, for every point, the nearest and second-nearest
// centroid under approximate distances R~ = fl32(sum_q fma((x_q - c~_q)^2)) (c~ = fp32(c)),
// together with a rigorous bound |R~ - rho^2| <= eps(R~) on the rounding error (rho the exact
// real distance).  When R~_2 - eps(R~_2) > R~_1 + eps(R~_1) (with 1e-12 relative slack for the
// fp64 evaluation), the fp32 nearest is provably the unique exact argmin of the fp64 scan
// (R8) -- its exact fp64 distance is computed and the point is done; lo =
// sqrt(R~_2 - eps(R~_2)) is a valid lower bound of the distance to every other centroid.
// Ambiguous points are queued for the exact scan (assign3_kernel).  Bound (u = 2^-24,
// eta = 2^-149 for subnormal results, C_m = max_c ||c||):
//   ||e|| <= u rho + theta,  theta = u (1+u) C_m + 3 eta sqrt(d)   (e = computed - exact diffs)
//   |sum diff~^2 - rho^2| <= (2u + u^2) rho^2 + 2 theta (1+u) rho + theta^2
//   |R~ - sum diff~^2| <= gamma_d sum diff~^2,  gamma_d = d u / (1 - d u)
//   => |R~ - rho^2| <= A rho^2 + B rho + C, solved for rho <= rho_max(R~).
// (The expanded form ||x||^2 + ||c||^2 - 2 x.c halves the arithmetic but its error scales
// with ||x|| ||c|| instead of rho^2: measured on configs[3] features it left up to 44 % of
// the points undecided, against < 0.003 % here.)
// ---------------------------------------------------------------------------
struct ScreenBound {
  double A, B, C;
  __device__ ScreenBound(double cm, int d) {
    const double u = 0x1p-24, eta = 0x1p-149;
    const double g = d * u / (1.0 - d * u);
    const double theta = u * (1.0 + u) * cm * 1.0001 + 4.0 * eta * sqrt((double)d);
    A = g + (1.0 + g) * (2.0 * u + u * u);
    B = 2.0 * (1.0 + g) * (1.0 + u) * theta;
    C = (1.0 + g) * theta * theta + (d + 1) * eta;
  }
  __device__ double eps(double R) const {
    const double rho = (B + sqrt(B * B + 4.0 * (1.0 - A) * (R + C))) / (2.0 * (1.0 - A));
    return (A * rho * rho + B * rho + C) * (1.0 + 1e-6) + 1e-300;
  }
};

__device__ __forceinline__ uint64_t pack2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}

// fp32 copy of the centroids and C_m = max_c ||c|| (rounded up)
__global__ void centroid_prep_kernel(const double* __restrict__ C, int k, int d, float* __restrict__ Cf,
                                     double* __restrict__ cm) {
  __shared__ double sh[256];
  double m = 0.0;
  for (int c = threadIdx.x; c < k; c += blockDim.x) {
    double s2 = 0.0;
    for (int q = 0; q < d; ++q) {
      const double v = C[(size_t)c * d + q];
      Cf[(size_t)c * d + q] = (float)v;
      s2 += v * v;
    }
    m = fmax(m, sqrt(s2));
  }
  sh[threadIdx.x] = m;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sh[threadIdx.x] = fmax(sh[threadIdx.x], sh[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *cm = sh[0] * (1.0 + 1e-9);
}

constexpr int kSPT = 128;              // points per block of the screen
constexpr int kSLX = kSPT + 4;         // padded leading dimensions (16-byte aligned rows)
constexpr int kSLC = kAT + 2;         // (8-byte aligned rows; staging writes at most 2-way conflicted)

template <int NBUF>
__global__ void __launch_bounds__(256, 3) assign_screen_kernel(const float* __restrict__ F, int64_t n, int d,
                                                            const double* __restrict__ C,
                                                            const float* __restrict__ Cf,
                                                            const double* __restrict__ cm, int k,
                                                            const int32_t* __restrict__ list,
                                                            const int* __restrict__ list_len,
                                                            int32_t* __restrict__ lab, double* __restrict__ dmin,
                                                            double* __restrict__ lo, int32_t* __restrict__ amb,
                                                            int* __restrict__ amb_len) {
  constexpr int nbuf = NBUF;
  // 128 points x 64-centroid tiles per block; thread (ty, tx) owns points ty*8 .. ty*8+7 and
  // the centroid pairs (2tx, 2tx+1), (2tx+32, 2tx+33) of a tile: 16 packed accumulators.
  // Packed fp32x2 arithmetic (FADD2/FFMA2: two IEEE round-to-nearest lanes per instruction,
  // the same rounding as scalar code, so the bound above holds lane by lane).
  extern __shared__ float smf[];
  float* sX = smf;                                    // [d][kSLX]
  float* sCb = smf + (size_t)d * kSLX;                // nbuf x [d][kSLC]: centroid tiles (double-
                                                      // buffered unless that costs the 3rd block/SM)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int tx = tid & 15, ty = tid >> 4;
  const int64_t m = list ? (int64_t)*list_len : n;
  const int64_t p0 = (int64_t)blockIdx.x * kSPT;
  if (p0 >= m) return;
  // the tile's point indices first (one load per thread, not one dependent load per row)
  __shared__ int s_gi[kSPT];
  if (tid < kSPT) {
    const int64_t pi = p0 + tid;
    s_gi[tid] = pi < m ? (list ? list[pi] : static_cast<int>(pi)) : -1;
  }
  __syncthreads();
  // staging: a warp takes one row (coalesced 4-byte cp.async, lanes along the row, stored
  // down the column), every copy of the tile in flight at once
  for (int row = warp; row < kSPT; row += 8) {
    const int64_t gi = s_gi[row];
    for (int q = lane; q < d; q += 32) {
      float* dst = sX + (size_t)q * kSLX + row;
      if (gi >= 0) {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
                     "l"(F + gi * d + q) : "memory");
      } else {
        *dst = 0.f;
      }
    }
  }
  float best[8], second[8];
  int bidx[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { best[i] = INFINITY; second[i] = INFINITY; bidx[i] = -1; }
  // centroid tile t goes to buffer t & 1; tile t+1 is requested before tile t is computed
  auto stage_c = [&](int c0, float* buf) {
    const int kt = min(kAT, k - c0);
    for (int cc = warp; cc < kAT; cc += 8)
      for (int q = lane; q < d; q += 32) {
        float* dst = buf + (size_t)q * kSLC + cc;
        if (cc < kt) {
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
                       "l"(Cf + (size_t)(c0 + cc) * d + q) : "memory");
        } else {
          *dst = 0.f;
        }
      }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  stage_c(0, sCb);   // (commits the point tile's copies too)
  for (int c0 = 0, t = 0; c0 < k; c0 += kAT, ++t) {
    const int kt = min(kAT, k - c0);
    float* sC = sCb + (size_t)(nbuf == 2 ? (t & 1) : 0) * d * kSLC;
    if (nbuf == 2 && c0 + kAT < k) {
      stage_c(c0 + kAT, sCb + (size_t)((t + 1) & 1) * d * kSLC);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    uint64_t acc[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) { acc[i][0] = 0ull; acc[i][1] = 0ull; }
    if (kt > 32) {
#pragma unroll 4
      for (int q = 0; q < d; ++q) {
        const float4 xa = *reinterpret_cast<const float4*>(sX + (size_t)q * kSLX + ty * 8);
        const float4 xb = *reinterpret_cast<const float4*>(sX + (size_t)q * kSLX + ty * 8 + 4);
        const uint64_t c01 = *reinterpret_cast<const uint64_t*>(sC + (size_t)q * kSLC + 2 * tx);
        const uint64_t c23 = *reinterpret_cast<const uint64_t*>(sC + (size_t)q * kSLC + 2 * tx + 32);
        const float xs[8] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint64_t xv = pack2(xs[i], xs[i]);
          uint64_t d0, d1;
          asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d0) : "l"(xv), "l"(c01));
          asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d1) : "l"(xv), "l"(c23));
          asm("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(acc[i][0]) : "l"(d0));
          asm("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(acc[i][1]) : "l"(d1));
        }
      }
    } else {
      // tail tile of <= 32 centroids (e.g. k = 200 = 3 x 64 + 8): the upper half of the
      // tile is padding, skip its arithmetic
#pragma unroll 4
      for (int q = 0; q < d; ++q) {
        const float4 xa = *reinterpret_cast<const float4*>(sX + (size_t)q * kSLX + ty * 8);
        const float4 xb = *reinterpret_cast<const float4*>(sX + (size_t)q * kSLX + ty * 8 + 4);
        const uint64_t c01 = *reinterpret_cast<const uint64_t*>(sC + (size_t)q * kSLC + 2 * tx);
        const float xs[8] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint64_t xv = pack2(xs[i], xs[i]);
          uint64_t d0;
          asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d0) : "l"(xv), "l"(c01));
          asm("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(acc[i][0]) : "l"(d0));
        }
      }
    }
    __syncthreads();   // every warp is done reading sC before the next request refills it
    if (nbuf == 1 && c0 + kAT < k) stage_c(c0 + kAT, sCb);
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int l = 0; l < 2; ++l) {
        const int cidx = 2 * tx + 32 * h + l;   // ascending per thread
        if (cidx < kt) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float v = __uint_as_float((unsigned)(acc[i][h] >> (32 * l)));
            if (v < best[i]) { second[i] = best[i]; best[i] = v; bidx[i] = c0 + cidx; }
            else if (v < second[i]) second[i] = v;
          }
        }
      }
  }
  // (R~, index) lexicographic min over the 16 threads of each point row, second best merged
#pragma unroll
  for (int i = 0; i < 8; ++i) {
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) {
      const float ob = __shfl_xor_sync(0xffffffffu, best[i], o);
      const float os = __shfl_xor_sync(0xffffffffu, second[i], o);
      const int oi = __shfl_xor_sync(0xffffffffu, bidx[i], o);
      const bool take = (oi >= 0) && (bidx[i] < 0 || ob < best[i] || (ob == best[i] && oi < bidx[i]));
      const float loser = take ? best[i] : ob;
      second[i] = fminf(fminf(second[i], os), loser);
      if (take) { best[i] = ob; bidx[i] = oi; }
    }
  }
  // thread tx < 8 of row ty handles point ty*8 + tx
  const int i = tx & 7;
  float bv = best[0], sv = second[0];
  int bl = bidx[0];
#pragma unroll
  for (int ii = 1; ii < 8; ++ii) if (ii == i) { bv = best[ii]; sv = second[ii]; bl = bidx[ii]; }
  const int col = ty * 8 + i;
  const int64_t pi = p0 + col;
  if (tx < 8 && pi < m) {
    const int64_t gi = s_gi[col];
    const ScreenBound sb(*cm, d);
    bool unique = false;
    double low = 0.0;
    if (bl >= 0 && isfinite(bv)) {
      const double r1 = bv, r2 = sv;
      const double up = (r1 + sb.eps(r1)) * (1.0 + 1e-12);
      low = isinf(r2) ? (double)INFINITY : (r2 - sb.eps(r2)) * (1.0 - 1e-12);
      unique = low > up;
    }
    if (unique) {
      const double* c = C + (size_t)bl * d;
      double acc = 0.0;
      for (int q = 0; q < d; ++q) {
        const double diff = __dsub_rn((double)sX[(size_t)q * kSLX + col], c[q]);
        acc = __dadd_rn(acc, __dmul_rn(diff, diff));
      }
      lab[gi] = bl;
      dmin[gi] = acc;
      lo[gi] = sqrt(low);
    } else {
      amb[atomicAdd(amb_len, 1)] = static_cast<int32_t>(gi);
    }
  }
}

// Pruning test (Hamerly): the centroids moved by at most dmax since lo_i (a lower bound
// of the distance to every centroid but the assigned one) was computed.  The exact
// squared distance to the assigned centroid is computed with the scan's arithmetic; if
// its root is below the decremented bound (with a 1e-9 relative margin for rounding),
// the assigned centroid is the unique argmin and the point keeps it -- the labels are the
// ones a full scan would produce.  Otherwise the point is queued for a full scan.
__global__ void __launch_bounds__(kSP) check_kernel(const float* __restrict__ F, int64_t n, int d,
                                                    const double* __restrict__ C, const int32_t* __restrict__ old_lab,
                                                    const double* __restrict__ dmax, int32_t* __restrict__ lab,
                                                    double* __restrict__ dmin, double* __restrict__ lo,
                                                    int32_t* __restrict__ list, int* __restrict__ list_len) {
  extern __shared__ unsigned char smk[];
  float* sx = reinterpret_cast<float*>(smk);
  const int64_t p0 = (int64_t)blockIdx.x * kSP;
  const bool v4 = rows_v4(F, d);
  stage_rows(F, n, d, p0, sx, v4);
  __syncthreads();
  const double dm = *dmax;
  const int64_t i = p0 + threadIdx.x;
  const bool in = i < n;
  bool keep = true;
  if (in) {
    const int a = old_lab[i];
    const double acc = row_dist(sx + threadIdx.x * rows_ld(v4, d), C + (size_t)a * d, d, v4);
    const double l = lo[i] - dm;
    lo[i] = l;
    keep = sqrt(acc) * (1.0 + 1e-9) < l * (1.0 - 1e-9);
    if (keep) {
      lab[i] = a;
      dmin[i] = acc;
    }
  }
  const unsigned need = __ballot_sync(0xffffffffu, !keep);
  if (!keep) {
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(need) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(list_len, __popc(need));
    base = __shfl_sync(need, base, leader);
    list[base + __popc(need & ((1u << lane) - 1))] = static_cast<int32_t>(i);
  }
}

// Bound-only pruning test of the screened path (Hamerly's upper bound, no feature read):
// u_i bounds the distance from x_i to its centroid -- sqrt(dmin_i) (1 + 1e-12) when dmin_i is
// exact for the current label (u_i < 0 or NaN: the last assignment computed it), else the
// carried bound -- and the centroid moved by at most shift[a] since, so
//   ||x_i - c_a_new|| <= (u_i + shift[a]) (1 + 1e-12) =: ub.
// lo_i (a lower bound of the distance to every other centroid) drops by dmax as in
// check_kernel.  If ub (1 + 1e-9) < (lo_i - dmax)(1 - 1e-9) the assigned centroid is the
// unique nearest (the margins cover the fp64 evaluation of R8, as in check_kernel): the point
// keeps its label and carries ub, its dmin is left stale (final_dmin_kernel recomputes the
// stale ones once the restart ends).  Otherwise it is queued for the screen, which computes
// its exact dmin (u_i = -1 marks that).
__global__ void __launch_bounds__(256) check_bound_kernel(int64_t n, const int32_t* __restrict__ old_lab,
                                                          const double* __restrict__ dmin, double* __restrict__ u,
                                                          double* __restrict__ lo, const double* __restrict__ shift,
                                                          const double* __restrict__ dmax, int32_t* __restrict__ lab,
                                                          int32_t* __restrict__ list, int* __restrict__ list_len) {
  const double dm = *dmax;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = base + threadIdx.x;
    bool keep = true;
    if (i < n) {
      const int a = old_lab[i];
      const double ui = u[i];
      const double b0 = ui >= 0.0 ? ui : sqrt(dmin[i]) * (1.0 + 1e-12);
      const double ub = (b0 + shift[a]) * (1.0 + 1e-12);
      const double l = lo[i] - dm;
      lo[i] = l;
      keep = ub * (1.0 + 1e-9) < l * (1.0 - 1e-9);
      if (keep) {
        lab[i] = a;
        u[i] = ub;
      } else {
        u[i] = -1.0;
      }
    }
    const unsigned need = __ballot_sync(0xffffffffu, !keep);
    if (!keep) {
      const int lane = threadIdx.x & 31;
      const int leader = __ffs(need) - 1;
      int b = 0;
      if (lane == leader) b = atomicAdd(list_len, __popc(need));
      b = __shfl_sync(need, b, leader);
      list[b + __popc(need & ((1u << lane) - 1))] = static_cast<int32_t>(i);
    }
  }
}

// The exact R8 distances of the points whose dmin is stale (u_i >= 0: kept by
// check_bound_kernel since their last exact distance) to their final centroid, staged rows as
// in check_kernel; then the restart's inertia is summed again (inertia_parts_kernel).
__global__ void __launch_bounds__(kSP) final_dmin_kernel(const float* __restrict__ F, int64_t n, int d,
                                                         const double* __restrict__ C,
                                                         const int32_t* __restrict__ lab, const double* __restrict__ u,
                                                         double* __restrict__ dmin) {
  extern __shared__ unsigned char smk[];
  float* sx = reinterpret_cast<float*>(smk);
  __shared__ int s_any;
  const int64_t p0 = (int64_t)blockIdx.x * kSP;
  const int64_t i = p0 + threadIdx.x;
  const bool stale = i < n && u[i] >= 0.0;
  if (threadIdx.x == 0) s_any = 0;
  __syncthreads();
  if (stale) s_any = 1;
  __syncthreads();
  if (!s_any) return;
  const bool v4 = rows_v4(F, d);
  stage_rows(F, n, d, p0, sx, v4);
  __syncthreads();
  if (stale) dmin[i] = row_dist(sx + threadIdx.x * rows_ld(v4, d), C + (size_t)lab[i] * d, d, v4);
}

// inertia partials with assign_stats_kernel's summation order (grid nstat x 256: each thread
// sums its grid-stride points in order, then the same block tree), so the total is the one a
// pass with exact distances throughout would give
__global__ void __launch_bounds__(256) inertia_parts_kernel(const double* __restrict__ dmin, int64_t n,
                                                            double* __restrict__ part_inertia) {
  double inertia = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
    const int64_t i = base + threadIdx.x;
    if (i < n) inertia += dmin[i];
  }
  __shared__ double sh[256];
  sh[threadIdx.x] = inertia;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part_inertia[blockIdx.x] = sh[0];
}

// Per-assignment statistics: cluster sizes, the list of changed points with the histogram of
// their old and new labels, and per-block inertia partials.  Grid-stride blocks keep both
// histograms in shared memory (k <= kHistMax) and flush k atomics per block at the end: a
// per-warp global atomic per distinct label (~30 per warp for random labels, k >= 100) cost
// 1.9 ms per assignment on configs[4].  Inertia: each thread sums its points in order, then a
// fixed block tree -- deterministic.
constexpr int kHistMax = 4096;
__global__ void __launch_bounds__(256) assign_stats_kernel(const int32_t* __restrict__ lab,
                                                           const int32_t* __restrict__ old_lab,
                                                           const double* __restrict__ dmin, int64_t n, int k,
                                                           int local,
                                                           double* __restrict__ part_inertia,
                                                           int* __restrict__ changed, unsigned* __restrict__ counts,
                                                           int32_t* __restrict__ chg_list,
                                                           unsigned* __restrict__ dcount) {
  extern __shared__ unsigned hist[];   // [2][k] when local (k <= kHistMax, blocks loop)
  unsigned* h_cnt = hist;
  unsigned* h_d = hist + (local ? k : 0);
  if (local)
    for (int c = threadIdx.x; c < 2 * k; c += blockDim.x) hist[c] = 0u;
  __syncthreads();
  unsigned* cnt_dst = local ? h_cnt : counts;
  unsigned* d_dst = local ? h_d : dcount;
  double inertia = 0.0;
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // (the loop bound is warp-uniform: every lane runs the same number of iterations)
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
    const int64_t i = base + threadIdx.x;
    const bool valid = i < n;
    const int bl = valid ? lab[i] : -1;
    if (valid) inertia += dmin[i];
    const int ol = (valid && old_lab) ? old_lab[i] : bl;
    const bool chg = valid && ol != bl;
    const unsigned peers = __match_any_sync(0xffffffffu, bl);
    if (valid && lane == __ffs(peers) - 1) atomicAdd(&cnt_dst[bl], (unsigned)__popc(peers));
    const unsigned cm = __ballot_sync(0xffffffffu, chg);
    if (cm) {
      const int leader = __ffs(cm) - 1;
      int b0 = 0;
      if (lane == leader) b0 = atomicAdd(changed, __popc(cm));
      b0 = __shfl_sync(0xffffffffu, b0, leader);
      if (chg) {
        chg_list[b0 + __popc(cm & ((1u << lane) - 1))] = static_cast<int32_t>(i);
        atomicAdd(&d_dst[bl], 1u);
        atomicAdd(&d_dst[ol], 1u);
      }
    }
  }
  __shared__ double sh[256];
  sh[threadIdx.x] = inertia;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part_inertia[blockIdx.x] = sh[0];
  if (local)
    for (int c = threadIdx.x; c < k; c += blockDim.x) {
      if (h_cnt[c]) atomicAdd(&counts[c], h_cnt[c]);
      if (h_d[c]) atomicAdd(&dcount[c], h_d[c]);
    }
}

// Centroid sums are kept as exact integers, so they can also be updated incrementally: the
// full recompute (plan, scatter, member sums) runs iff full_gate(); otherwise
// the changed points are filed +/- under their new / old clusters (scatter_any_kernel) and
// the member sums move their contributions between clusters.  The
// decision reads the device-side changed-label count (no host round trip).
__device__ __forceinline__ bool full_gate(const int* chg, int64_t thresh) {
  return chg == nullptr || (int64_t)*chg > thresh;
}

// members of cluster c land at perm[off[c] .. off[c+1]) (order inside a cluster is
// arbitrary; the exact integer sums below do not depend on it).  scatter_any_kernel (below)
// ranks a block's points per cluster in shared memory and reserves one slice per (block,
// cluster) with a single global atomic; this simple variant serves k > 6144.
__global__ void scatter_members_simple_kernel(const int32_t* __restrict__ lab, int64_t n,
                                              unsigned* __restrict__ cursor, const int64_t* __restrict__ off,
                                              int32_t* __restrict__ perm, const int* __restrict__ chg,
                                              int64_t thresh) {
  if (!full_gate(chg, thresh)) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = lab[i];
    perm[off[c] + atomicAdd(&cursor[c], 1u)] = static_cast<int32_t>(i);
  }
}

// Device-side plan of the member sums (no host round trip): cluster offsets off[0..k]
// (exclusive scan of the histogram) and the first work item item0[0..k] of each cluster
// (work items of <= chunk members, ascending clusters); item0[k] = number of items.
__global__ void zero_acc_kernel(unsigned long long* __restrict__ acc4, int64_t cnt, const int* __restrict__ chg,
                                int64_t thresh) {
  if (!full_gate(chg, thresh)) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x)
    acc4[i] = 0ull;
}

// (full recompute: histogram of the labels; incremental: histogram of the changed points'
// old and new labels)
// Zeroing for the next steps rides along (one launch instead of several memsets): the
// histograms, changed-label slot and queue lengths the next assignment accumulates into, the
// scatter cursors, and (full recompute, small k d) the limb accumulators.
struct PlanZero {
  int* changed_slot;          // next assignment's changed-label counter
  unsigned* counts_next;      // [k] next assignment's histogram
  unsigned* dcount_next;      // [k] next assignment's changed-point histogram
  unsigned* cursor;           // [k] scatter cursors
  int* len;                   // pruning / ambiguous queue lengths ([0] and [2])
  unsigned long long* acc4;   // limb accumulators (zeroed here iff acc_n > 0 and full recompute)
  int64_t acc_n;
  double* cm;                 // max centroid norm / largest shift, merged by the finalize kernel
  double* dmax;
};

__global__ void __launch_bounds__(256) plan_members_kernel(const unsigned* __restrict__ counts_full,
                                                           const unsigned* __restrict__ counts_delta, int k,
                                                           int64_t chunk, int64_t* __restrict__ off,
                                                           int32_t* __restrict__ item0, int* __restrict__ total_items,
                                                           const int* __restrict__ chg, int64_t thresh, PlanZero z) {
  const bool full = full_gate(chg, thresh);
  const unsigned* __restrict__ counts = full ? counts_full : counts_delta;
  for (int c = threadIdx.x; c < k; c += blockDim.x) {
    if (z.counts_next) z.counts_next[c] = 0u;
    if (z.dcount_next) z.dcount_next[c] = 0u;
    if (z.cursor) z.cursor[c] = 0u;
  }
  if (threadIdx.x == 0) {
    if (z.changed_slot) *z.changed_slot = 0;
    if (z.len) { z.len[0] = 0; z.len[2] = 0; }
    if (z.cm) *z.cm = 0.0;
    if (z.dmax) *z.dmax = 0.0;
  }
  if (full && z.acc_n > 0)
    for (int64_t e = threadIdx.x; e < z.acc_n; e += blockDim.x) z.acc4[e] = 0ull;
  __shared__ long long s_cnt[256];
  __shared__ int s_ni[256];
  __shared__ long long carry_off;
  __shared__ int carry_it;
  const int tid = threadIdx.x;
  if (tid == 0) { carry_off = 0; carry_it = 0; }
  __syncthreads();
  for (int base = 0; base < k; base += 256) {
    const int c = base + tid;
    const long long cnt = c < k ? (long long)counts[c] : 0;
    const int ni = (int)((cnt + chunk - 1) / chunk);
    s_cnt[tid] = cnt;
    s_ni[tid] = ni;
    __syncthreads();
    for (int o = 1; o < 256; o <<= 1) {   // inclusive Hillis-Steele scans
      const long long a = tid >= o ? s_cnt[tid - o] : 0;
      const int b = tid >= o ? s_ni[tid - o] : 0;
      __syncthreads();
      s_cnt[tid] += a;
      s_ni[tid] += b;
      __syncthreads();
    }
    if (c < k) {
      off[c] = carry_off + s_cnt[tid] - cnt;   // exclusive
      item0[c] = carry_it + s_ni[tid] - ni;
    }
    __syncthreads();
    if (tid == 255) { carry_off += s_cnt[255]; carry_it += s_ni[255]; }
    __syncthreads();
  }
  if (tid == 0) {
    off[k] = carry_off;
    item0[k] = carry_it;
    *total_items = carry_it;
  }
}

__device__ __forceinline__ void add_limbs(unsigned long long* a, unsigned __int128 u) {
#pragma unroll
  for (int l = 0; l < 4; ++l) {
    const unsigned long long limb = (unsigned long long)(u >> (32 * l)) & 0xffffffffull;
    if (limb) atomicAdd(a + l, limb);
  }
}

// Exact member sums: block w takes work item w -- cluster c (item0[c] <= w < item0[c+1],
// binary search), members [off[c] + j chunk, min(off[c+1], off[c] + (j+1) chunk)) with
// j = w - item0[c].  Thread (slot, dim q) accumulates x * 2^shift exactly in a 128-bit integer,
// the block reduces its slots, and the block sum of each dim is added, as four 32-bit limbs,
// to the cluster's 64-bit limb accumulators acc[c][q][0..3] (integer atomics: exact and order
// independent; < 2^32 items keep every limb sum below 2^64).
__global__ void member_sum_kernel(const float* __restrict__ F, int d, const int32_t* __restrict__ perm,
                                  const int64_t* __restrict__ off, const int32_t* __restrict__ item0, int k,
                                  int64_t chunk, const int* __restrict__ total_items, int shift,
                                  unsigned long long* __restrict__ acc4 /* [k][d][4] */) {
  extern __shared__ unsigned long long red2[];   // [slots][d][2]
  __shared__ int s_c;
  const int w = blockIdx.x;
  if (w >= *total_items) return;
  if (threadIdx.x == 0) {
    int lo = 0, hi = k;   // largest c with item0[c] <= w
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (item0[mid] <= w) lo = mid; else hi = mid;
    }
    s_c = lo;
  }
  __syncthreads();
  const int c = s_c;
  const int64_t wsb = off[c] + (int64_t)(w - item0[c]) * chunk;
  const int64_t web = min(off[c + 1], wsb + chunk);
  const int slots = blockDim.x / d;
  const int j = threadIdx.x / d, q = threadIdx.x - j * d;
  __int128 acc = 0;
  if (j < slots) {
    int64_t m = wsb + j;
    // entry bit 31: subtract (incremental update); eight independent gathers in flight
    for (; m + 7 * slots < web; m += 8 * slots) {
      float x[8];
      uint32_t e[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        e[u] = static_cast<uint32_t>(perm[m + u * slots]);
        x[u] = F[(int64_t)(e[u] & 0x7fffffffu) * d + q];
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const __int128 v = to_fixed(x[u], shift);
        acc += (e[u] >> 31) ? -v : v;
      }
    }
    for (; m < web; m += slots) {
      const uint32_t e = static_cast<uint32_t>(perm[m]);
      const __int128 v = to_fixed(F[(int64_t)(e & 0x7fffffffu) * d + q], shift);
      acc += (e >> 31) ? -v : v;
    }
  }
  if (j < slots) {
    red2[((size_t)j * d + q) * 2] = (unsigned long long)acc;
    red2[((size_t)j * d + q) * 2 + 1] = (unsigned long long)(acc >> 64);
  }
  __syncthreads();
  if (threadIdx.x < d) {
    __int128 sum = 0;
    for (int jj = 0; jj < slots; ++jj) {
      const unsigned long long lo = red2[((size_t)jj * d + threadIdx.x) * 2];
      const unsigned long long hi = red2[((size_t)jj * d + threadIdx.x) * 2 + 1];
      sum += (__int128)(((unsigned __int128)hi << 64) | lo);
    }
    add_limbs(acc4 + ((size_t)c * d + threadIdx.x) * 4, (unsigned __int128)sum);
  }
}

// Full or incremental scatter in one launch (device-side choice, block-uniform branch):
// full -> counting sort of all points by label (blocks of per_block points, per-block
// shared-memory ranks, one global atomic per (block, cluster)), incremental -> the changed points filed +/- (scatter_delta_kernel).
__global__ void scatter_any_kernel(const int32_t* __restrict__ lab, int64_t n, int k, int64_t per_block,
                                   unsigned* __restrict__ cursor, const int64_t* __restrict__ off,
                                   int32_t* __restrict__ perm, const int32_t* __restrict__ chg_list,
                                   const int* __restrict__ chg, const int32_t* __restrict__ prev, int64_t thresh) {
  extern __shared__ unsigned hist[];   // [k] local counts, then [k] bases
  if (full_gate(chg, thresh)) {
    unsigned* base = hist + k;
    const int64_t a = blockIdx.x * per_block;
    if (a >= n) return;
    const int64_t b = min(n, a + per_block);
    for (int c = threadIdx.x; c < k; c += blockDim.x) hist[c] = 0;
    __syncthreads();
    for (int64_t i = a + threadIdx.x; i < b; i += blockDim.x) atomicAdd(&hist[lab[i]], 1u);
    __syncthreads();
    for (int c = threadIdx.x; c < k; c += blockDim.x) {
      base[c] = hist[c] ? atomicAdd(&cursor[c], hist[c]) : 0u;
      hist[c] = 0;
    }
    __syncthreads();
    for (int64_t i = a + threadIdx.x; i < b; i += blockDim.x) {
      const int c = lab[i];
      perm[off[c] + base[c] + atomicAdd(&hist[c], 1u)] = static_cast<int32_t>(i);
    }
  } else {
    const int m = *chg;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) {
      const int32_t i = chg_list[j];
      const int bl = lab[i], al = prev[i];
      perm[off[bl] + atomicAdd(&cursor[bl], 1u)] = i;
      perm[off[al] + atomicAdd(&cursor[al], 1u)] = static_cast<int32_t>(static_cast<uint32_t>(i) | 0x80000000u);
    }
  }
}

// Incremental exact update: every changed point (old label a -> new label b) is listed
// under cluster b with sign + and under cluster a with sign - (bit 31 of the entry); the
// member sums then move its fixed-point image between the clusters exactly.
__global__ void scatter_delta_kernel(const int32_t* __restrict__ chg_list, const int* __restrict__ chg,
                                     const int32_t* __restrict__ prev, const int32_t* __restrict__ cur,
                                     unsigned* __restrict__ cursor, const int64_t* __restrict__ off,
                                     int32_t* __restrict__ perm, int64_t thresh) {
  if (full_gate(chg, thresh)) return;
  const int m = *chg;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) {
    const int32_t i = chg_list[j];
    const int b = cur[i], a = prev[i];
    perm[off[b] + atomicAdd(&cursor[b], 1u)] = i;
    perm[off[a] + atomicAdd(&cursor[a], 1u)] = static_cast<int32_t>(static_cast<uint32_t>(i) | 0x80000000u);
  }
}

// C[c][q] = correctly rounded (cluster sum) / count; empty clusters keep C.  The sum is
// sum_l acc[c][q][l] 2^(32 l) mod 2^128, read as a signed 128-bit integer; the limbs are
// rewritten in canonical form (each < 2^32), so the next update starts from one add per limb.
// One block per centroid, which also produces what the next assignment's bounds need (no
// separate passes): the fp32 copy Cf for the screen, max_c ||c|| (cm) and the largest
// centroid shift max_c ||c_new - c_old|| (dmax, Hamerly), both rounded up by 1e-9 and merged
// with atomicMax on their bit patterns (non-negative doubles order as integers); cm and dmax
// were zeroed by the plan kernel.
__global__ void __launch_bounds__(256) member_finalize_kernel(unsigned long long* __restrict__ acc4,
                                                              const unsigned* __restrict__ counts, int k, int d,
                                                              int shift, double* __restrict__ C,
                                                              float* __restrict__ Cf, double* __restrict__ cm,
                                                              double* __restrict__ dmax, double* __restrict__ shifts) {
  __shared__ double s_n[256], s_d[256];
  const int c = blockIdx.x;
  const unsigned cnt = counts[c];
  double n2 = 0.0, d2 = 0.0;
  for (int q = threadIdx.x; q < d; q += blockDim.x) {
    const int64_t e = (int64_t)c * d + q;
    unsigned long long* a = acc4 + e * 4;
    unsigned __int128 u = 0;
#pragma unroll
    for (int l = 0; l < 4; ++l) u += (unsigned __int128)a[l] << (32 * l);
#pragma unroll
    for (int l = 0; l < 4; ++l) a[l] = (unsigned long long)(u >> (32 * l)) & 0xffffffffull;
    const double old = C[e];
    const double v = cnt ? fixed_to_double((__int128)u, shift) / (double)cnt : old;
    C[e] = v;
    if (Cf) Cf[e] = (float)v;
    n2 += v * v;
    d2 += (v - old) * (v - old);
  }
  if (!cm && !dmax) return;   // (small problems: no screen, no pruning)
  s_n[threadIdx.x] = n2;
  s_d[threadIdx.x] = d2;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) { s_n[threadIdx.x] += s_n[threadIdx.x + o]; s_d[threadIdx.x] += s_d[threadIdx.x + o]; }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (cm) atomicMax(reinterpret_cast<unsigned long long*>(cm),
                      (unsigned long long)__double_as_longlong(sqrt(s_n[0]) * (1.0 + 1e-9)));
    if (dmax) {
      const double sh = sqrt(s_d[0]) * (1.0 + 1e-9) + 1e-300;
      atomicMax(reinterpret_cast<unsigned long long*>(dmax), (unsigned long long)__double_as_longlong(sh));
      if (shifts) shifts[c] = sh;   // this centroid's move (bound-only pruning test)
    }
  }
}

int num_sms_current() {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

}  // namespace

int normalize_rows_f32(float* F, int64_t n, int d, cudaStream_t s) {
  normalize_rows_kernel<<<num_sms_current() * 8, kB, 0, s>>>(F, n, d);
  SC_CUDA_TRY(cudaGetLastError());
  return SC_OK;
}

// ---------------------------------------------------------------------------
// k-means driver
// ---------------------------------------------------------------------------
namespace {
struct KmResult {
  double inertia = INFINITY;
  int iters = 0;
  int r = -1;
  std::vector<double> C;
};
}  // namespace

// Process-wide pool of pinned int buffers (never returned to the driver).
struct PinnedSlot {
  int* p = nullptr;
  size_t n = 0;
  static std::mutex& mu() { static std::mutex m; return m; }
  static std::vector<std::pair<int*, size_t>>& free_list() {
    static std::vector<std::pair<int*, size_t>> f;
    return f;
  }
  int acquire(size_t want) {
    {
      std::lock_guard<std::mutex> lk(mu());
      auto& f = free_list();
      for (size_t i = 0; i < f.size(); ++i)
        if (f[i].second >= want) {
          p = f[i].first;
          n = f[i].second;
          f.erase(f.begin() + (long)i);
          return SC_OK;
        }
    }
    SC_CUDA_TRY(cudaMallocHost(&p, sizeof(int) * want));
    n = want;
    return SC_OK;
  }
  ~PinnedSlot() {
    if (!p) return;
    std::lock_guard<std::mutex> lk(mu());
    free_list().emplace_back(p, n);
  }
};

// Restarts r0, r0 + rstep, ... < restarts on stream s; the best of them (lowest inertia,
// ties -> lowest r) goes to *res and its labels to labels_dev.
static int kmeans_worker(const float* F, int64_t n, int d, int k, int r0, int rstep, int restarts, int max_iter,
                         uint64_t seed, const double* uniforms_host, int32_t* labels_dev, KmResult* res,
                         cudaStream_t s, Coll* coll = nullptr, int64_t row_off = 0, int64_t n_global = -1,
                         const double* init_C = nullptr) {
  // init_C (device, restarts x k x d): the k-means++ seeds of every restart, already drawn by
  // seed_batch (kmeans_run); the worker then only runs Lloyd
  // coll != nullptr: distributed over the ranks of a row partition (kmeans_run_dist) -- the
  // same kernels on the local rows; the fixed-point scale, the changed-label counts, the exact
  // member sums and counts, the inertia and the k-means++ draws are reduced over the ranks
  if (n_global < 0) n_global = n;
  const int sms = num_sms_current();
  const int grid = sms * 8;
  const int G = std::min(sms * 2, 1024);                  // k-means++ range blocks (<= kSel)
  const int64_t chunk = (n + G - 1) / G;
  // workspace
  // assignment: 64 points x 64-centroid tiles per block, fp64 [d][64] tiles of both
  const int smem_assign = (int)(sizeof(double) * 2 * (size_t)d * kAT);
  if (smem_assign > 200 * 1024) return fail(SC_ERR_ARG, "sc_kmeans: d must be <= 200");
  const int64_t nblk = (n + kAT - 1) / kAT;
  const int64_t list_grid = std::min<int64_t>(nblk, (int64_t)sms * 4);   // list-mode scans: grid-stride
  constexpr int64_t kChunk = 512;    // members per exact-sum work item
  const int64_t max_items = 2 * n / kChunk + k + 1;   // (incremental lists: 2 entries per changed point)
  PoolBuf b_lab, b_new, b_d2, b_C, b_cnt, b_cur, b_off, b_perm, b_items, b_part, b_psum, b_misc;
  SC_TRY(b_lab.ensure(sizeof(int32_t) * n, s));
  SC_TRY(b_new.ensure(sizeof(int32_t) * n, s));
  SC_TRY(b_d2.ensure(sizeof(double) * n, s));
  SC_TRY(b_C.ensure(sizeof(double) * k * d, s));
  SC_TRY(b_cnt.ensure(sizeof(unsigned) * 2 * k, s));   // histograms, by assignment parity
  SC_TRY(b_cur.ensure(sizeof(unsigned) * k, s));
  SC_TRY(b_off.ensure(sizeof(int64_t) * (k + 1), s));
  SC_TRY(b_perm.ensure(sizeof(int32_t) * 2 * n, s));
  SC_TRY(b_items.ensure(sizeof(int32_t) * (k + 1), s));
  SC_TRY(b_psum.ensure(sizeof(unsigned long long) * 4 * (size_t)k * d, s));
  const int64_t nstat = std::min<int64_t>((n + 255) / 256, (int64_t)sms * 8);   // assign_stats_kernel grid
  // shared-memory histograms only when the blocks loop over several 256-point groups (small
  // problems keep one group per block and direct atomics)
  const bool stats_local = k <= kHistMax && n > nstat * 256;
  SC_TRY(b_part.ensure(sizeof(double) * std::max<int64_t>(std::max<int64_t>(grid, G), std::max(nblk, nstat)), s));
  PoolBuf b_dmin, b_lo, b_list, b_len, b_dmax;
  SC_TRY(b_dmin.ensure(sizeof(double) * n, s));
  SC_TRY(b_lo.ensure(sizeof(double) * n, s));
  SC_TRY(b_list.ensure(sizeof(int32_t) * n, s));
  SC_TRY(b_len.ensure(16, s));   // [0] pruning queue length, [1] member work items, [2] ambiguous
  SC_TRY(b_dmax.ensure(16, s));
  // bound-only pruning of the screened path: distance upper bounds (u < 0: dmin exact) and
  // the centroids' moves of the last update
  PoolBuf b_u, b_shift;
  SC_TRY(b_u.ensure(sizeof(double) * n, s));
  SC_TRY(b_shift.ensure(sizeof(double) * (k + 1), s));
  PoolBuf b_chg, b_near, b_gap;
  SC_TRY(b_chg.ensure(sizeof(int) * (max_iter + 2), s));
  SC_TRY(b_near.ensure(sizeof(int32_t) * n, s));     // k-means++: nearest seed per point
  SC_TRY(b_gap.ensure(sizeof(double) * (k + 1), s));  // half distances new seed -> earlier seeds
  // screened assignment: fp32 centroids, C_m, queue of the points the screen cannot decide
  PoolBuf b_Cf, b_amb, b_chgl, b_dcnt;
  SC_TRY(b_chgl.ensure(sizeof(int32_t) * n, s));
  SC_TRY(b_dcnt.ensure(sizeof(unsigned) * 2 * k, s));
  SC_TRY(b_Cf.ensure(sizeof(float) * (size_t)k * d + 64, s));
  SC_TRY(b_amb.ensure(sizeof(int32_t) * n, s));
  float* d_Cf = b_Cf.as<float>();
  double* d_cm = reinterpret_cast<double*>(b_Cf.as<char>() + ((sizeof(float) * (size_t)k * d + 15) / 16) * 16);
  // pinned landing slots for the changed-label counts, from a process-wide pool (worker
  // threads are short-lived: a per-thread cudaMallocHost / cudaFreeHost pair per call
  // synchronises the device and showed up as 0.5-0.9 s outliers in the stability scan)
  PinnedSlot pin;
  SC_TRY(pin.acquire(2 * ((size_t)max_iter + 2)));
  int* h_chg = pin.p;
  int* h_rescan = pin.p + max_iter + 2;   // pruning-queue length per iteration (-1: no check run)
  cudaEvent_t ev_chg[2];
  SC_CUDA_TRY(cudaEventCreateWithFlags(&ev_chg[0], cudaEventDisableTiming));
  SC_CUDA_TRY(cudaEventCreateWithFlags(&ev_chg[1], cudaEventDisableTiming));
  struct EvGuard { cudaEvent_t* e; ~EvGuard() { cudaEventDestroy(e[0]); cudaEventDestroy(e[1]); } } ev_guard{ev_chg};
  SC_TRY(b_misc.ensure(64, s));
  PoolBuf b_gcnt, b_sall;   // distributed: global member counts, per-rank D^2 totals (+ 1 scratch)
  if (coll) {
    SC_TRY(b_gcnt.ensure(sizeof(unsigned) * k, s));
    SC_TRY(b_sall.ensure(sizeof(double) * (coll->world + 1), s));
  }
  int32_t* lab = b_lab.as<int32_t>();
  int32_t* nw = b_new.as<int32_t>();
  double* C = b_C.as<double>();
  int* changed = b_misc.as<int>();
  unsigned* absmax = reinterpret_cast<unsigned*>(b_misc.as<char>() + 32);

  // fixed-point scale from the largest |feature|
  SC_CUDA_TRY(cudaMemsetAsync(absmax, 0, sizeof(unsigned), s));
  absmax_bits_kernel<<<grid, kB, 0, s>>>(F, n * d, absmax);
  SC_CUDA_TRY(cudaGetLastError());
  if (coll) SC_TRY(coll->max_u32(absmax, 1, s));   // one fixed-point scale on every rank
  unsigned amax_bits = 0;
  SC_CUDA_TRY(cudaMemcpyAsync(&amax_bits, absmax, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
  SC_CUDA_TRY(cudaStreamSynchronize(s));
  float amax;
  std::memcpy(&amax, &amax_bits, sizeof(float));
  if (!std::isfinite(amax)) return fail(SC_ERR_ARG, "features contain inf/nan");
  int E = 0;
  if (amax > 0.0f) { std::frexp((double)amax, &E); }   // amax < 2^E
  const int shift = 100 - E;   // |x| 2^shift < 2^100; sums of < 2^25 members fit 2^125

  // exact scan: the centroid tile width 16 NC with the fewest padded columns (ties: wider)
  int nc_best = 4;
  {
    int best_cols = 1 << 30;
    for (int nc : {4, 2, 1}) {
      const int tw = 16 * nc, cols = (k + tw - 1) / tw * tw;
      if (cols < best_cols) { best_cols = cols; nc_best = nc; }
    }
  }
  auto assign3 = nc_best == 4 ? assign3_kernel<4> : nc_best == 2 ? assign3_kernel<2> : assign3_kernel<1>;
  SC_TRY(smem_attr_at_least(reinterpret_cast<const void*>(assign3), smem_assign));
  // the screens' ambiguous points: warp-per-point scan when the centroids fit in shared memory
  // (env SC_KMEANS_AMB_WARP=0: the tile kernel)
  const int smem_amb = (int)(sizeof(double) * ((size_t)k * d + 8 * (size_t)d));
  const bool amb_direct = k <= kAmbK && smem_amb <= 100 * 1024 &&
                          !(std::getenv("SC_KMEANS_AMB_WARP") && std::atoi(std::getenv("SC_KMEANS_AMB_WARP")) == 0);
  int64_t amb_grid = 1;
  if (amb_direct) {
    SC_TRY(smem_attr_at_least(reinterpret_cast<const void*>(amb_scan_kernel), smem_amb));
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, amb_scan_kernel, 256, smem_amb);
    amb_grid = (int64_t)sms * std::max(1, occ);
  }
  // double-buffered centroid tiles unless that drops the screen below 3 blocks per SM (d > ~70)
  int smem_sm = 0, cur_dev = 0;
  cudaGetDevice(&cur_dev);
  cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, cur_dev);
  const auto screen_bytes = [&](int nb) { return (int)(sizeof(float) * (size_t)d * (kSLX + nb * kSLC)); };
  const int screen_nbuf = 3 * (screen_bytes(2) + 512 + 1024) <= smem_sm ? 2 : 1;
  const int smem_screen = screen_bytes(screen_nbuf);
  SC_TRY(smem_attr_at_least(reinterpret_cast<const void*>(screen_nbuf == 2 ? assign_screen_kernel<2> : assign_screen_kernel<1>), smem_screen));
  // the screen pays off when the exact scan is expensive (env SC_KMEANS_SCREEN=0 disables it);
  // threshold measured on the configs[2] stability scan (k-means 0.57 s at 2^27, 0.47 s at 3e7
  // and 1e7: 10^5 x 48 features, k = 10..30); the Hamerly check follows the same size rule
  // (0.475 -> 0.466 s)
  const double screen_min = std::getenv("SC_KMEANS_SCREEN_MIN") ? std::atof(std::getenv("SC_KMEANS_SCREEN_MIN"))
                                                                : 3.0e7;
  const bool screen = (double)n * k * d >= screen_min && !(std::getenv("SC_KMEANS_SCREEN") && std::atoi(std::getenv("SC_KMEANS_SCREEN")) == 0);
  const int smem_rows = (int)(sizeof(float) * kSP * (d + 4));   // (row stride d + 4 or d + 1)
  const int smem_d2 = smem_rows + (int)(sizeof(double) * d);
  SC_TRY(smem_attr_at_least(reinterpret_cast<const void*>(check_kernel), smem_rows));
  SC_TRY(smem_attr_at_least(reinterpret_cast<const void*>(d2_update_kernel), smem_d2));
  SC_TRY(smem_attr_at_least(reinterpret_cast<const void*>(d2_update_skip_kernel), smem_d2));

  // tensor-core screen (sc_kmeans_tc.cu) for the assignments after a restart's first (env
  // SC_KMEANS_TC=0: the fp32 screen throughout)
  const bool use_tc = screen && tc_screen_supported(k, d);
  TcWork tcw;
  // Lloyd assignment of every point; host receives inertia (fixed-order sum of block
  // partials), the number of changed labels and the label histogram
  // Hamerly pruning pays off when a full assignment is expensive; small problems (many of
  // them in a stability scan) are launch-bound and take the plain full scan
  const double prune_min = std::getenv("SC_KMEANS_PRUNE_MIN") ? std::atof(std::getenv("SC_KMEANS_PRUNE_MIN"))
                                                              : 3.0e7;
  const bool prune = (double)n * k * d >= prune_min;
  // the screened path prunes with bounds only (check_bound_kernel: no feature reads; the
  // stale distances are recomputed once per restart); env SC_KMEANS_BOUND=0: exact check
  const bool bound_check = screen && prune && !(std::getenv("SC_KMEANS_BOUND") && std::atoi(std::getenv("SC_KMEANS_BOUND")) == 0);
  if (bound_check) SC_TRY(smem_attr_at_least(reinterpret_cast<const void*>(final_dmin_kernel), smem_rows));
  // Lloyd assignment of every point, no host synchronisation: labels, exact dmin, the
  // number of changed labels into changed_dev[slot] and the label histogram (device);
  // block partials of the inertia in b_part
  int* changed_dev = b_chg.as<int>();
  const bool trace_len = std::getenv("SC_KMEANS_TRACE") != nullptr;
  // (the counters an assignment accumulates into -- changed_dev[slot], the histograms of
  // parity slot & 1, the queue lengths -- were zeroed by the preceding update's plan kernel,
  // or before the first assignment of a restart)
  auto cnt_of = [&](int slot) { return b_cnt.as<unsigned>() + (size_t)(slot & 1) * k; };
  auto dcnt_of = [&](int slot) { return b_dcnt.as<unsigned>() + (size_t)(slot & 1) * k; };
  auto assign_all = [&](int32_t* out_lab, const int32_t* old, int slot, bool try_check) -> int {
    if (screen) {
      // fp32 screen + exact verification of every point (or of the pruning queue), exact
      // fp64 scan of the points it cannot decide
      const bool pruned = old && prune && try_check;
      int* amb_len = b_len.as<int>() + 2;
      if (pruned) {
        if (bound_check) {
          check_bound_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)sms * 16), 256, 0, s>>>(
              n, old, b_dmin.as<double>(), b_u.as<double>(), b_lo.as<double>(), b_shift.as<double>(),
              b_dmax.as<double>(), out_lab, b_list.as<int32_t>(), b_len.as<int>());
        } else {
          check_kernel<<<(unsigned)((n + kSP - 1) / kSP), kSP, smem_rows, s>>>(
              F, n, d, C, old, b_dmax.as<double>(), out_lab, b_dmin.as<double>(), b_lo.as<double>(),
              b_list.as<int32_t>(), b_len.as<int>());
        }
        SC_CUDA_TRY(cudaGetLastError());
      } else if (bound_check) {
        // every point's dmin is recomputed by this assignment: no carried bounds
        SC_CUDA_TRY(cudaMemsetAsync(b_u.ptr, 0xff, sizeof(double) * n, s));
      }
      if (!old) {   // first assignment of a restart; later ones get Cf, cm from the finalize kernel
        centroid_prep_kernel<<<1, 256, 0, s>>>(C, k, d, d_Cf, d_cm);
        SC_CUDA_TRY(cudaGetLastError());
      }
      if (old && use_tc) {
        // tensor-core screen in coordinates centred on each point's current centroid
        SC_TRY(tc_screen(F, n, d, C, d_Cf, d_cm, k, old, pruned ? b_list.as<int32_t>() : nullptr,
                         pruned ? b_len.as<int>() : nullptr, out_lab, b_dmin.as<double>(), b_lo.as<double>(),
                         b_amb.as<int32_t>(), amb_len, tcw, s));
      } else {
        (screen_nbuf == 2 ? assign_screen_kernel<2> : assign_screen_kernel<1>)<<<(unsigned)((n + kSPT - 1) / kSPT),
                                                                                 256, smem_screen, s>>>(
            F, n, d, C, d_Cf, d_cm, k, pruned ? b_list.as<int32_t>() : nullptr, pruned ? b_len.as<int>() : nullptr,
            out_lab, b_dmin.as<double>(), b_lo.as<double>(), b_amb.as<int32_t>(), amb_len);
      }
      SC_CUDA_TRY(cudaGetLastError());
      if (amb_direct) {
        amb_scan_kernel<<<(unsigned)amb_grid, 256, smem_amb, s>>>(F, d, C, k, b_amb.as<int32_t>(), amb_len, out_lab,
                                                                   b_dmin.as<double>(), b_lo.as<double>());
      } else {
        assign3<<<(unsigned)list_grid, 256, smem_assign, s>>>(F, n, d, C, k, b_amb.as<int32_t>(), amb_len, out_lab,
                                                               b_dmin.as<double>(), b_lo.as<double>());
      }
      if (trace_len) {
        int h_len[3] = {0, 0, 0};
        SC_CUDA_TRY(cudaMemcpyAsync(h_len, b_len.ptr, sizeof(h_len), cudaMemcpyDeviceToHost, s));
        SC_CUDA_TRY(cudaStreamSynchronize(s));
        std::fprintf(stderr, "[sc_kmeans] iteration %d: %d rescanned, %d ambiguous of %lld\n", slot,
                     pruned ? h_len[0] : (int)n, h_len[2], (long long)n);
      }
    } else if (!old || !prune) {
      // full scan of every point (the first assignment of a restart also sets the bounds lo)
      assign3<<<(unsigned)nblk, 256, smem_assign, s>>>(F, n, d, C, k, nullptr, nullptr, out_lab,
                                                             b_dmin.as<double>(), b_lo.as<double>());
    } else {
      // Hamerly pruning: points whose assigned centroid is provably still the unique
      // nearest keep it; the rest are queued and fully rescanned
      check_kernel<<<(unsigned)((n + kSP - 1) / kSP), kSP, smem_rows, s>>>(
          F, n, d, C, old, b_dmax.as<double>(), out_lab, b_dmin.as<double>(), b_lo.as<double>(),
          b_list.as<int32_t>(), b_len.as<int>());
      SC_CUDA_TRY(cudaGetLastError());
      assign3<<<(unsigned)list_grid, 256, smem_assign, s>>>(F, n, d, C, k, b_list.as<int32_t>(), b_len.as<int>(),
                                                             out_lab, b_dmin.as<double>(), b_lo.as<double>());
      if (trace_len) {
        int h_len = 0;
        SC_CUDA_TRY(cudaMemcpyAsync(&h_len, b_len.ptr, sizeof(int), cudaMemcpyDeviceToHost, s));
        SC_CUDA_TRY(cudaStreamSynchronize(s));
        std::fprintf(stderr, "[sc_kmeans] iteration %d: %d of %lld points rescanned\n", slot, h_len, (long long)n);
      }
    }
    SC_CUDA_TRY(cudaGetLastError());
    assign_stats_kernel<<<(unsigned)nstat, 256, stats_local ? sizeof(unsigned) * 2 * k : 0, s>>>(
        out_lab, old, b_dmin.as<double>(), n, k, stats_local ? 1 : 0, b_part.as<double>(),
                                                       changed_dev + slot, cnt_of(slot),
                                                       b_chgl.as<int32_t>(), dcnt_of(slot));
    SC_CUDA_TRY(cudaGetLastError());
    if (coll) SC_TRY(coll->sum_i32(changed_dev + slot, 1, s));   // labels changed on any rank
    return SC_OK;
  };
  auto read_inertia = [&](double* inertia) -> int {
    std::vector<double> part(nstat);
    SC_CUDA_TRY(cudaMemcpyAsync(part.data(), b_part.as<double>(), sizeof(double) * nstat, cudaMemcpyDeviceToHost, s));
    SC_CUDA_TRY(cudaStreamSynchronize(s));
    double tot = 0.0;
    for (double v : part) tot += v;   // fixed order: deterministic
    if (coll) {   // + the other ranks' totals, in rank order
      double* dv = b_sall.as<double>() + coll->world;
      SC_CUDA_TRY(cudaMemcpyAsync(dv, &tot, sizeof(double), cudaMemcpyHostToDevice, s));
      SC_TRY(coll->sum_f64(dv, 1, s));
      SC_CUDA_TRY(cudaMemcpyAsync(&tot, dv, sizeof(double), cudaMemcpyDeviceToHost, s));
      SC_CUDA_TRY(cudaStreamSynchronize(s));
    }
    *inertia = tot;
    return SC_OK;
  };

  // centroids <- member means of the labels `cur` (histogram on the device): members grouped
  // by cluster (counting sort), exact 128-bit fixed-point member sums, one rounding
  int64_t* d_off = b_off.as<int64_t>();
  int32_t* d_item0 = b_items.as<int32_t>();
  int* d_total = b_len.as<int>() + 1;
  // full recompute when more than n/4 labels changed (or no previous sums), else incremental
  // (2 gathered rows per changed point against n)
  const int64_t delta_thresh = n / 4;
  // update(it): centroids from the labels of assignment it-1 (histograms of parity it-1);
  // its plan kernel zeroes what assignment it accumulates into
  const int64_t acc_elems = 4 * (int64_t)k * d;
  auto update = [&](const int32_t* cur, const int32_t* prev, const int* chg, int it) -> int {
    if (!prev) chg = nullptr;
    const bool big_acc = acc_elems > 65536;
    if (big_acc) {
      zero_acc_kernel<<<std::max(1, std::min(grid, (int)((acc_elems + kB - 1) / kB))), kB, 0, s>>>(
          b_psum.as<unsigned long long>(), acc_elems, chg, delta_thresh);
      SC_CUDA_TRY(cudaGetLastError());
    }
    const PlanZero z{changed_dev + it, cnt_of(it), dcnt_of(it), b_cur.as<unsigned>(), b_len.as<int>(),
                     b_psum.as<unsigned long long>(), big_acc ? 0 : acc_elems, screen ? d_cm : nullptr,
                     prune ? b_dmax.as<double>() : nullptr};
    plan_members_kernel<<<1, 256, 0, s>>>(cnt_of(it - 1), dcnt_of(it - 1), k, kChunk, d_off, d_item0, d_total, chg,
                                          delta_thresh, z);
    SC_CUDA_TRY(cudaGetLastError());
    if (k <= 6144) {
      const int64_t per_block = std::max<int64_t>(4096, (n + grid - 1) / grid);
      const int64_t sgrid = std::max<int64_t>((n + per_block - 1) / per_block, prev ? grid : 1);
      scatter_any_kernel<<<(unsigned)sgrid, kB, sizeof(unsigned) * 2 * k, s>>>(
          cur, n, k, per_block, b_cur.as<unsigned>(), d_off, b_perm.as<int32_t>(), b_chgl.as<int32_t>(), chg, prev,
          delta_thresh);
    } else {
      scatter_members_simple_kernel<<<grid, kB, 0, s>>>(cur, n, b_cur.as<unsigned>(), d_off, b_perm.as<int32_t>(),
                                                        chg, delta_thresh);
      if (prev)
        scatter_delta_kernel<<<grid, kB, 0, s>>>(b_chgl.as<int32_t>(), chg, prev, cur, b_cur.as<unsigned>(), d_off,
                                                 b_perm.as<int32_t>(), delta_thresh);
    }
    SC_CUDA_TRY(cudaGetLastError());
    const int slots = std::max(1, 256 / d);
    member_sum_kernel<<<(unsigned)max_items, slots * d, sizeof(unsigned long long) * 2 * slots * d, s>>>(
        F, d, b_perm.as<int32_t>(), d_off, d_item0, k, kChunk, d_total, shift, b_psum.as<unsigned long long>());
    SC_CUDA_TRY(cudaGetLastError());
    const unsigned* counts = cnt_of(it - 1);
    if (coll) {
      // exact integer sums over the ranks (order independent), member counts likewise
      SC_TRY(coll->sum_u64(b_psum.as<unsigned long long>(), (size_t)acc_elems, s));
      SC_CUDA_TRY(cudaMemcpyAsync(b_gcnt.ptr, counts, sizeof(unsigned) * k, cudaMemcpyDeviceToDevice, s));
      SC_TRY(coll->sum_u32(b_gcnt.as<unsigned>(), (size_t)k, s));
      counts = b_gcnt.as<unsigned>();
    }
    {
      // bounds wanted: 256 threads (power of two for the block reduction); else one warp-multiple
      const bool bounds = screen || prune;
      const int fin_threads = bounds ? 256 : std::min(256, (d + 31) / 32 * 32);
      member_finalize_kernel<<<(unsigned)k, fin_threads, 0, s>>>(
          b_psum.as<unsigned long long>(), counts, k, d, shift, C, screen ? d_Cf : nullptr,
          screen ? d_cm : nullptr, prune ? b_dmax.as<double>() : nullptr,
          (screen && prune) ? b_shift.as<double>() : nullptr);
    }
    SC_CUDA_TRY(cudaGetLastError());
    return SC_OK;
  };

  double best_inertia = INFINITY;
  int best_r = -1, best_it = 0;
  std::vector<double> best_C((size_t)k * d);
  std::vector<double> u(k);
  const bool trace = std::getenv("SC_KMEANS_TRACE") != nullptr;
  auto now = [] { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
  double t_seed = 0.0, t_lloyd = 0.0, t_mark = now();
  for (int r = r0; r < restarts; r += rstep) {
    if (trace) t_mark = now();
    for (int t = 0; t < k; ++t)
      u[t] = uniforms_host ? uniforms_host[(size_t)r * k + t] : uniform_host(seed, 1, (uint64_t)r * k + t);
    // ---- k-means++ seeding (device-resident: block sums, then one selection kernel per draw)
    int64_t idx = std::min<int64_t>((int64_t)std::floor(u[0] * n_global), n_global - 1);
    if (init_C) {
      SC_CUDA_TRY(cudaMemcpyAsync(C, init_C + (size_t)r * k * d, sizeof(double) * k * d, cudaMemcpyDeviceToDevice, s));
    } else if (!coll) {
      row_to_centroid_kernel<<<1, 128, 0, s>>>(F, idx, d, C);
    } else {
      row_or_zero_kernel<<<1, 128, 0, s>>>(F, (idx >= row_off && idx < row_off + n) ? idx - row_off : -1, d, C);
      SC_TRY(coll->sum_f64(C, (size_t)d, s));
    }
    if (!init_C) {
    d2_update_kernel<<<(unsigned)((n + kSP - 1) / kSP), kSP, smem_d2, s>>>(F, n, d, C, b_d2.as<double>(), 1,
                                                                          b_near.as<int32_t>());
    SC_CUDA_TRY(cudaGetLastError());
    }
    for (int t = 1; t < k && !init_C; ++t) {
      range_sums_kernel<<<G, kB, 0, s>>>(b_d2.as<double>(), n, chunk, b_part.as<double>());
      if (!coll) {
        seed_select_kernel<<<1, kSel, 0, s>>>(b_part.as<double>(), G, b_d2.as<double>(), n, chunk, u[t], F, d,
                                            C + (size_t)t * d, t, b_gap.as<double>());
      } else {
        SC_CUDA_TRY(cudaMemsetAsync(b_sall.ptr, 0, sizeof(double) * coll->world, s));
        local_total_kernel<<<1, kSel, 0, s>>>(b_part.as<double>(), G, coll->rank, b_sall.as<double>());
        SC_TRY(coll->sum_f64(b_sall.as<double>(), (size_t)coll->world, s));
        seed_select_dist_kernel<<<1, kSel, 0, s>>>(b_part.as<double>(), G, b_d2.as<double>(), n, chunk, u[t],
                                                 b_sall.as<double>(), DistDraw{coll->rank, coll->world, row_off,
                                                                               n_global},
                                                 F, d, C + (size_t)t * d);
        SC_TRY(coll->sum_f64(C + (size_t)t * d, (size_t)d, s));
        half_gap_kernel<<<1, 256, 0, s>>>(C, d, t, b_gap.as<double>());
      }
      d2_update_skip_kernel<<<(unsigned)((n + kSP - 1) / kSP), kSP, smem_d2, s>>>(
          F, n, d, C + (size_t)t * d, t, b_gap.as<double>(), b_d2.as<double>(), b_near.as<int32_t>());
      SC_CUDA_TRY(cudaGetLastError());
    }
    // ---- Lloyd.  Iterations are issued without waiting; the changed-label count of
    // iteration it-1 is read (pinned copy + event) while iteration it runs.  Once an
    // assignment repeats, further iterations are idempotent (same labels -> same exact
    // means -> same labels), so the one issued speculatively changes nothing but time.
    if (trace) { SC_CUDA_TRY(cudaStreamSynchronize(s)); t_seed += now() - t_mark; t_mark = now(); }
    // counters of the first assignment (later ones are zeroed by the update plan kernels)
    SC_CUDA_TRY(cudaMemsetAsync(changed_dev, 0, sizeof(int), s));
    SC_CUDA_TRY(cudaMemsetAsync(b_cnt.ptr, 0, sizeof(unsigned) * k, s));
    SC_CUDA_TRY(cudaMemsetAsync(b_dcnt.ptr, 0, sizeof(unsigned) * k, s));
    SC_CUDA_TRY(cudaMemsetAsync(b_len.ptr, 0, 3 * sizeof(int), s));
    SC_TRY(assign_all(lab, nullptr, 0, false));
    int it = 0, conv = -1;
    // With the screen on, the Hamerly check is only worth its extra pass over the features
    // while it keeps most points: it is skipped once it queued >= 60 % of them (known with
    // one iteration of lag) and re-tried every 8th iteration.
    bool use_check = true;
    int last_check = 0;
    for (it = 1; it <= max_iter; ++it) {
      const bool try_check = !screen || use_check || it - last_check >= 8;
      if (try_check) last_check = it;
      // (distributed: full recompute every iteration -- the incremental update would keep
      // per-rank running sums apart from the reduced ones)
      SC_TRY(update(lab, (it >= 2 && !coll) ? nw : nullptr, changed_dev + (it - 1), it));
      SC_TRY(assign_all(nw, lab, it, try_check));
      SC_CUDA_TRY(cudaMemcpyAsync(h_chg + it, changed_dev + it, sizeof(int), cudaMemcpyDeviceToHost, s));
      if (screen && try_check)
        SC_CUDA_TRY(cudaMemcpyAsync(h_rescan + it, b_len.ptr, sizeof(int), cudaMemcpyDeviceToHost, s));
      else
        h_rescan[it] = -1;
      SC_CUDA_TRY(cudaEventRecord(ev_chg[it & 1], s));
      std::swap(lab, nw);
      if (it >= 2) {
        SC_CUDA_TRY(cudaEventSynchronize(ev_chg[(it - 1) & 1]));
        if (h_chg[it - 1] == 0) { conv = it - 1; break; }
        if (h_rescan[it - 1] >= 0) use_check = (double)h_rescan[it - 1] < 0.6 * (double)n;
        if (trace_len) std::fprintf(stderr, "[sc_kmeans] iteration %d: %d labels changed\n", it - 1, h_chg[it - 1]);
      }
    }
    if (conv < 0) {
      SC_CUDA_TRY(cudaStreamSynchronize(s));
      const int last = std::min(it, max_iter);
      conv = h_chg[last] == 0 ? last : max_iter;
      // (a run that never converges ends at max_iter, like the oracle)
    }
    it = conv;
    if (bound_check) {
      // the stale distances of the points the bound-only test kept, then the inertia again
      final_dmin_kernel<<<(unsigned)((n + kSP - 1) / kSP), kSP, smem_rows, s>>>(F, n, d, C, lab, b_u.as<double>(),
                                                                               b_dmin.as<double>());
      inertia_parts_kernel<<<(unsigned)nstat, 256, 0, s>>>(b_dmin.as<double>(), n, b_part.as<double>());
      SC_CUDA_TRY(cudaGetLastError());
    }
    double inertia = 0.0;
    SC_TRY(read_inertia(&inertia));
    if (trace) {
      t_lloyd += now() - t_mark;
      std::fprintf(stderr, "[sc_kmeans] restart %d: seeding %.4f s, lloyd %.4f s (%d iters)\n", r, t_seed, t_lloyd, it);
    }
    if (inertia < best_inertia) {
      best_inertia = inertia;
      best_r = r;
      best_it = it;
      SC_CUDA_TRY(cudaMemcpyAsync(labels_dev, lab, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, s));
      SC_CUDA_TRY(cudaMemcpyAsync(best_C.data(), C, sizeof(double) * k * d, cudaMemcpyDeviceToHost, s));
      SC_CUDA_TRY(cudaStreamSynchronize(s));
    }
  }
  res->inertia = best_inertia;
  res->iters = best_it;
  res->r = best_r;
  res->C = best_C;
  return SC_OK;
}

int kmeans_run_dist(const float* F, int64_t n_local, int64_t row_off, int64_t n_global, int d, int k, int restarts,
                    int max_iter, uint64_t seed, const double* uniforms_host, int32_t* labels_dev,
                    double* centroids_host, double* inertia_out, int* iters_out, int* best_out, Coll* coll,
                    cudaStream_t s) {
  // restarts one after another (every rank issues the same collectives in the same order)
  KmResult res;
  SC_TRY(kmeans_worker(F, n_local, d, k, 0, 1, restarts, max_iter, seed, uniforms_host, labels_dev, &res, s, coll,
                       row_off, n_global));
  if (res.r < 0) return fail(SC_ERR_ARG, "k-means produced no finite inertia");
  if (centroids_host) std::memcpy(centroids_host, res.C.data(), sizeof(double) * k * d);
  if (inertia_out) *inertia_out = res.inertia;
  if (iters_out) *iters_out = res.iters;
  if (best_out) *best_out = res.r;
  return SC_OK;
}

// k-means++ seeds of restarts [0, restarts) drawn together (the kernels above), into C_all
// (device, restarts x k x d).  Same uniforms, chunking and arithmetic as kmeans_worker's
// per-restart seeding, so the seeds are identical; batches of up to kSeedBatch restarts.
constexpr int kSeedBatch = 16;
static int seed_batch(const float* F, int64_t n, int d, int k, int restarts, uint64_t seed,
                      const double* uniforms_host, double* C_all, cudaStream_t s) {
  const int sms = num_sms_current();
  const int G = std::min(sms * 2, 1024);                  // as kmeans_worker
  const int64_t chunk = (n + G - 1) / G;
  const int64_t cstride = (int64_t)k * d;
  const int nb = std::min(restarts, kSeedBatch);
  PoolBuf b_d2, b_near, b_gap, b_part, b_u;
  SC_TRY(b_d2.ensure(sizeof(double) * (size_t)nb * n, s));
  SC_TRY(b_near.ensure(sizeof(int32_t) * (size_t)nb * n, s));
  SC_TRY(b_gap.ensure(sizeof(double) * (size_t)nb * (k + 1), s));
  SC_TRY(b_part.ensure(sizeof(double) * (size_t)nb * G, s));
  SC_TRY(b_u.ensure(sizeof(double) * (size_t)nb * k, s));
  const size_t smem = sizeof(double) * (size_t)nb * d + sizeof(float) * kSP * (size_t)(d + 4);
  SC_TRY(smem_attr_at_least(reinterpret_cast<const void*>(d2_first_batch_kernel), (int)smem));
  SC_TRY(smem_attr_at_least(reinterpret_cast<const void*>(d2_skip_batch_kernel), (int)smem));
  std::vector<double> u((size_t)nb * k);
  for (int r0 = 0; r0 < restarts; r0 += nb) {
    const int nr = std::min(nb, restarts - r0);
    for (int r = 0; r < nr; ++r)
      for (int t = 0; t < k; ++t)
        u[(size_t)r * k + t] = uniforms_host ? uniforms_host[(size_t)(r0 + r) * k + t]
                                             : uniform_host(seed, 1, (uint64_t)(r0 + r) * k + t);
    SC_CUDA_TRY(cudaMemcpyAsync(b_u.ptr, u.data(), sizeof(double) * (size_t)nr * k, cudaMemcpyHostToDevice, s));
    double* Cb = C_all + (size_t)r0 * cstride;
    for (int r = 0; r < nr; ++r) {
      const int64_t idx = std::min<int64_t>((int64_t)std::floor(u[(size_t)r * k] * n), n - 1);
      row_to_centroid_kernel<<<1, 128, 0, s>>>(F, idx, d, Cb + (size_t)r * cstride);
    }
    const unsigned pb = (unsigned)((n + kSP - 1) / kSP);
    d2_first_batch_kernel<<<pb, kSP, smem, s>>>(F, n, d, Cb, cstride, nr, b_d2.as<double>(), b_near.as<int32_t>());
    SC_CUDA_TRY(cudaGetLastError());
    for (int t = 1; t < k; ++t) {
      range_sums_batch_kernel<<<dim3(G, nr), kB, 0, s>>>(b_d2.as<double>(), n, chunk, G, b_part.as<double>());
      seed_select_batch_kernel<<<nr, kSel, 0, s>>>(b_part.as<double>(), G, b_d2.as<double>(), n, chunk,
                                                   b_u.as<double>(), k, F, d, Cb, cstride, t, b_gap.as<double>(),
                                                   k + 1);
      d2_skip_batch_kernel<<<pb, kSP, smem, s>>>(F, n, d, Cb, cstride, t, nr, b_gap.as<double>(), k + 1,
                                                 b_d2.as<double>(), b_near.as<int32_t>());
      SC_CUDA_TRY(cudaGetLastError());
    }
  }
  return SC_OK;
}

int kmeans_run(const float* F, int64_t n, int d, int k, int restarts, int max_iter, uint64_t seed,
               const double* uniforms_host, int32_t* labels_dev, double* centroids_host, double* inertia_out,
               int* iters_out, int* best_out, cudaStream_t s, int max_workers) {
  // Restarts are independent: large problems run them on worker threads, each with its own
  // stream and stream-ordered workspace (the pruned Lloyd phase and the k-means++ draws are
  // latency-bound, so concurrent restarts overlap); the winner is the same as in a sequential
  // loop (lowest inertia, ties -> lowest restart index).  Default 10 workers (configs[3]
  // sc_cluster k-means 0.293 s with 4, 0.284 s with 8, 0.273 s with 10); the stability scan,
  // which runs 8 problems at once, passes 4 (0.570 s vs 0.637 s with 10).
  static const int env_workers =
      std::getenv("SC_KMEANS_WORKERS") ? std::max(1, std::atoi(std::getenv("SC_KMEANS_WORKERS"))) : 10;
  if (max_workers <= 0) max_workers = env_workers;
  const int P = (restarts > 1 && (double)n * d >= 4.0e6) ? std::min(restarts, max_workers) : 1;
  std::vector<KmResult> res(P);
  if (P == 1) {
    SC_TRY(kmeans_worker(F, n, d, k, 0, 1, restarts, max_iter, seed, uniforms_host, labels_dev, &res[0], s));
  } else {
    int dev = 0;
    cudaGetDevice(&dev);
    // every restart's k-means++ seeds in one batched pass (env SC_KMEANS_SEED_BATCH=0: each
    // worker seeds its own restarts)
    PoolBuf b_init;
    const bool batch_seed = !(std::getenv("SC_KMEANS_SEED_BATCH") && std::atoi(std::getenv("SC_KMEANS_SEED_BATCH")) == 0);
    if (batch_seed) {
      SC_TRY(b_init.ensure(sizeof(double) * (size_t)restarts * k * d, s));
      SC_TRY(seed_batch(F, n, d, k, restarts, seed, uniforms_host, b_init.as<double>(), s));
    }
    const double* init_C = batch_seed ? b_init.as<double>() : nullptr;
    cudaEvent_t ready;
    SC_CUDA_TRY(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    SC_CUDA_TRY(cudaEventRecord(ready, s));
    std::vector<PoolBuf> labs(P);
    std::vector<cudaStream_t> streams(P, nullptr);
    std::vector<int> rcs(P, SC_OK);
    std::vector<std::string> msgs(P);
    std::vector<std::thread> pool;
    for (int w = 0; w < P; ++w) {
      pool.emplace_back([&, w]() {
        cudaSetDevice(dev);
        if (cudaStreamCreateWithFlags(&streams[w], cudaStreamNonBlocking) != cudaSuccess ||
            cudaStreamWaitEvent(streams[w], ready, 0) != cudaSuccess) {
          rcs[w] = SC_ERR_CUDA;
          msgs[w] = "worker stream creation failed";
          return;
        }
        int rc = labs[w].ensure(sizeof(int32_t) * n, streams[w]);
        if (rc == SC_OK)
          rc = kmeans_worker(F, n, d, k, w, P, restarts, max_iter, seed, uniforms_host, labs[w].as<int32_t>(),
                             &res[w], streams[w], nullptr, 0, -1, init_C);
        if (rc != SC_OK) {
          rcs[w] = rc;
          msgs[w] = sc_last_error();
        }
        cudaStreamSynchronize(streams[w]);
      });
    }
    for (auto& th : pool) th.join();
    cudaEventDestroy(ready);
    int win = -1;
    for (int w = 0; w < P; ++w) {
      if (rcs[w] != SC_OK) {
        for (int v = 0; v < P; ++v) {
          labs[v].release();
          if (streams[v]) cudaStreamDestroy(streams[v]);
        }
        return fail(rcs[w], "sc_kmeans worker: " + msgs[w]);
      }
      if (res[w].r >= 0 && (win < 0 || res[w].inertia < res[win].inertia ||
                            (res[w].inertia == res[win].inertia && res[w].r < res[win].r)))
        win = w;
    }
    if (win >= 0)
      SC_CUDA_TRY(cudaMemcpyAsync(labels_dev, labs[win].ptr, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, s));
    SC_CUDA_TRY(cudaStreamSynchronize(s));
    for (int w = 0; w < P; ++w) {
      labs[w].release();
      cudaStreamDestroy(streams[w]);
    }
    if (win > 0) std::swap(res[0], res[win]);
    else if (win < 0) res[0].r = -1;
  }
  if (res[0].r < 0) return fail(SC_ERR_ARG, "k-means produced no finite inertia");
  if (centroids_host) std::memcpy(centroids_host, res[0].C.data(), sizeof(double) * k * d);
  if (inertia_out) *inertia_out = res[0].inertia;
  if (iters_out) *iters_out = res[0].iters;
  if (best_out) *best_out = res[0].r;
  return SC_OK;
}

// ---------------------------------------------------------------------------
// adjusted Rand index
// ---------------------------------------------------------------------------
int ari_dev(const int32_t* a, const int32_t* b, int64_t n, double* out, cudaStream_t s) {
  const int sms = num_sms_current();
  DevBuf mm;
  SC_TRY(mm.ensure(4 * sizeof(int)));
  int init[4] = {INT_MAX, INT_MIN, INT_MAX, INT_MIN};
  SC_CUDA_TRY(cudaMemcpyAsync(mm.ptr, init, sizeof(init), cudaMemcpyHostToDevice, s));
  minmax_kernel<<<sms * 4, kB, 0, s>>>(a, n, mm.as<int>());
  minmax_kernel<<<sms * 4, kB, 0, s>>>(b, n, mm.as<int>() + 2);
  int h[4];
  SC_CUDA_TRY(cudaMemcpyAsync(h, mm.ptr, sizeof(h), cudaMemcpyDeviceToHost, s));
  SC_CUDA_TRY(cudaStreamSynchronize(s));
  if (h[0] < 0 || h[2] < 0) return fail(SC_ERR_ARG, "labels must be non-negative");
  const int ka = h[1] + 1, kb = h[3] + 1;
  if ((int64_t)ka * kb > (1 << 26)) return fail(SC_ERR_ARG, "too many labels for the contingency table");
  DevBuf t;
  SC_TRY(t.ensure(sizeof(unsigned long long) * ka * kb));
  SC_CUDA_TRY(cudaMemsetAsync(t.ptr, 0, sizeof(unsigned long long) * ka * kb, s));
  contingency_kernel<<<sms * 8, kB, 0, s>>>(a, b, n, ka, kb, t.as<unsigned long long>());
  SC_CUDA_TRY(cudaGetLastError());
  std::vector<unsigned long long> tab((size_t)ka * kb);
  SC_CUDA_TRY(cudaMemcpyAsync(tab.data(), t.ptr, sizeof(unsigned long long) * ka * kb, cudaMemcpyDeviceToHost, s));
  SC_CUDA_TRY(cudaStreamSynchronize(s));
  auto c2 = [](double x) { return x * (x - 1.0) / 2.0; };
  std::vector<double> ra(ka, 0.0), cb(kb, 0.0);
  double sum_ij = 0.0;
  int64_t nnz = 0;
  for (int i = 0; i < ka; ++i)
    for (int j = 0; j < kb; ++j) {
      const double v = (double)tab[(size_t)i * kb + j];
      if (v > 0) ++nnz;
      sum_ij += c2(v);
      ra[i] += v;
      cb[j] += v;
    }
  double sa = 0.0, sb = 0.0;
  int nra = 0, ncb = 0;
  for (double v : ra) { sa += c2(v); nra += v > 0; }
  for (double v : cb) { sb += c2(v); ncb += v > 0; }
  const double expected = n > 1 ? sa * sb / c2((double)n) : 0.0;
  const double denom = 0.5 * (sa + sb) - expected;
  if (denom == 0.0) *out = (nra == ncb && nnz == nra) ? 1.0 : 0.0;
  else *out = (sum_ij - expected) / denom;
  return SC_OK;
}

}  // namespace sc
