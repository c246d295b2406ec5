// Features -> clusters: row normalisation, k-means++ seeding, Lloyd iterations,
// adjusted Rand index.
//
// PAPER.md §2.2 step 4 (lines 109-113), §4.1 step 6 (lines 323-328): k-means with
// the Euclidean distance on the feature rows; §5: replicates.
// Decision arithmetic is fixed so that the result does not depend on thread
// scheduling (reading R8):
//   * distances: fp64, explicit differences, summed in ascending q with
//     __dsub_rn/__dmul_rn/__dadd_rn (no FMA contraction);
//   * centroid sums: exact fixed-point accumulation of the fp32 features in
//     three 38-bit limbs of 64-bit integer atomics (order independent), rounded
//     once to fp64 (= the correctly rounded sum), then divided by the count.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "sc_internal.cuh"

namespace sc {
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

__device__ __forceinline__ double dist2_row(const float* __restrict__ x, const double* __restrict__ c, int d) {
  double acc = 0.0;
  for (int q = 0; q < d; ++q) {
    const double diff = __dsub_rn((double)x[q], c[q]);
    acc = __dadd_rn(acc, __dmul_rn(diff, diff));
  }
  return acc;
}

// d2[i] = (first ? dist : min(d2[i], dist)) to centre c (device fp64 row)
__global__ void d2_update_kernel(const float* __restrict__ F, int64_t n, int d, const double* __restrict__ c,
                                 double* __restrict__ d2, int first) {
  extern __shared__ double sc_[];
  for (int q = threadIdx.x; q < d; q += blockDim.x) sc_[q] = c[q];
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = dist2_row(F + i * d, sc_, d);
    d2[i] = first ? v : fmin(d2[i], v);
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

// sequential scan of one range: first i with start + cumsum > target
__global__ void range_select_kernel(const double* __restrict__ v, int64_t b0, int64_t b1, double start,
                                    double target, int64_t* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double s = start;
  int64_t last_pos = -1;
  for (int64_t i = b0; i < b1; ++i) {
    s += v[i];
    if (v[i] > 0.0) last_pos = i;
    if (s > target) { *out = i; return; }
  }
  *out = last_pos >= 0 ? last_pos : b1 - 1;
}

__global__ void row_to_centroid_kernel(const float* __restrict__ F, int64_t idx, int d, double* __restrict__ c) {
  for (int q = threadIdx.x; q < d; q += blockDim.x) c[q] = (double)F[idx * d + q];
}

// assignment over a tile of centroids [c0, c0+kt); best (dist, label) kept in dmin/lab
__global__ void assign_kernel(const float* __restrict__ F, int64_t n, int d, const double* __restrict__ C,
                              int c0, int kt, int first_tile, int last_tile, int32_t* __restrict__ lab,
                              double* __restrict__ dmin, const int32_t* __restrict__ old_lab,
                              int* __restrict__ changed, double* __restrict__ part_inertia) {
  extern __shared__ double sC[];
  for (int e = threadIdx.x; e < kt * d; e += blockDim.x) sC[e] = C[(int64_t)c0 * d + e];
  __syncthreads();
  double inertia = 0.0;
  int nchg = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float* x = F + i * d;
    double best = first_tile ? INFINITY : dmin[i];
    int bl = first_tile ? -1 : lab[i];
    for (int c = 0; c < kt; ++c) {
      const double v = dist2_row(x, sC + c * d, d);
      if (v < best) { best = v; bl = c0 + c; }
    }
    if (bl < 0) bl = c0;   // all distances NaN/inf: deterministic fallback
    dmin[i] = best;
    lab[i] = bl;
    if (last_tile) {
      inertia += best;
      if (old_lab && old_lab[i] != bl) ++nchg;
    }
  }
  if (last_tile) {
    __shared__ double sh[kB];
    __shared__ int shc[kB];
    sh[threadIdx.x] = inertia;
    shc[threadIdx.x] = nchg;
    __syncthreads();
    for (int o = kB / 2; o > 0; o >>= 1) {
      if ((int)threadIdx.x < o) { sh[threadIdx.x] += sh[threadIdx.x + o]; shc[threadIdx.x] += shc[threadIdx.x + o]; }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      part_inertia[blockIdx.x] = sh[0];
      if (shc[0]) atomicAdd(changed, shc[0]);
    }
  }
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

constexpr int kLimb = 38;
constexpr unsigned long long kLimbMask = (1ull << kLimb) - 1ull;

// accumulate member sums for clusters [c0, c0+kt) into limbs[3][k][d] (global), counts[k]
__global__ void centroid_accum_kernel(const float* __restrict__ F, const int32_t* __restrict__ lab, int64_t n,
                                      int d, int c0, int kt, int shift, unsigned long long* __restrict__ limbs,
                                      int k, unsigned long long* __restrict__ counts, int do_counts) {
  extern __shared__ unsigned long long sl[];   // [3][kt*d] then counts[kt]
  const int slots = kt * d;
  for (int e = threadIdx.x; e < 3 * slots + kt; e += blockDim.x) sl[e] = 0ull;
  __syncthreads();
  const int64_t total = n * d;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / d;
    const int q = static_cast<int>(e - i * d);
    const int c = lab[i] - c0;
    if (c < 0 || c >= kt) continue;
    const __int128 v = to_fixed(F[e], shift);
    const unsigned long long l0 = (unsigned long long)(v & (__int128)kLimbMask);
    const __int128 v1 = v >> kLimb;
    const unsigned long long l1 = (unsigned long long)(v1 & (__int128)kLimbMask);
    const long long l2 = (long long)(v1 >> kLimb);
    const int slot = c * d + q;
    if (l0) atomicAdd(&sl[slot], l0);
    if (l1) atomicAdd(&sl[slots + slot], l1);
    if (l2) atomicAdd(&sl[2 * slots + slot], (unsigned long long)l2);
    if (do_counts && q == 0) atomicAdd(&sl[3 * slots + c], 1ull);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 3 * slots; e += blockDim.x) {
    const unsigned long long v = sl[e];
    if (v) {
      const int limb = e / slots, slot = e - limb * slots;
      atomicAdd(&limbs[(size_t)limb * k * d + (size_t)c0 * d + slot], v);
    }
  }
  if (do_counts)
    for (int c = threadIdx.x; c < kt; c += blockDim.x)
      if (sl[3 * slots + c]) atomicAdd(&counts[c0 + c], sl[3 * slots + c]);
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

__global__ void centroid_finalize_kernel(const unsigned long long* __restrict__ limbs,
                                         const unsigned long long* __restrict__ counts, int k, int d,
                                         int shift, double* __restrict__ C) {
  const int slots = k * d;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < slots; e += gridDim.x * blockDim.x) {
    const int c = e / d;
    const unsigned long long cnt = counts[c];
    if (cnt == 0) continue;   // empty cluster keeps its centre
    const __int128 S = (__int128)limbs[e] + ((__int128)limbs[slots + e] << kLimb) +
                       ((__int128)(long long)limbs[2 * slots + e] << (2 * kLimb));
    C[e] = fixed_to_double(S, shift) / (double)cnt;
  }
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
int kmeans_run(const float* F, int64_t n, int d, int k, int restarts, int max_iter, uint64_t seed,
               const double* uniforms_host, int32_t* labels_dev, double* centroids_host, double* inertia_out,
               int* iters_out, int* best_out, cudaStream_t s) {
  const int sms = num_sms_current();
  const int grid = sms * 8;
  const int G = sms * 2;                                  // k-means++ range blocks
  const int64_t chunk = (n + G - 1) / G;
  // workspace
  DevBuf b_lab, b_new, b_dmin, b_d2, b_C, b_limbs, b_cnt, b_part, b_misc;
  SC_TRY(b_lab.ensure(sizeof(int32_t) * n));
  SC_TRY(b_new.ensure(sizeof(int32_t) * n));
  SC_TRY(b_dmin.ensure(sizeof(double) * n));
  SC_TRY(b_d2.ensure(sizeof(double) * n));
  SC_TRY(b_C.ensure(sizeof(double) * k * d));
  SC_TRY(b_limbs.ensure(sizeof(unsigned long long) * 3 * k * d));
  SC_TRY(b_cnt.ensure(sizeof(unsigned long long) * k));
  SC_TRY(b_part.ensure(sizeof(double) * std::max(grid, G)));
  SC_TRY(b_misc.ensure(64));
  int32_t* lab = b_lab.as<int32_t>();
  int32_t* nw = b_new.as<int32_t>();
  double* C = b_C.as<double>();
  int* changed = b_misc.as<int>();
  int64_t* sel = reinterpret_cast<int64_t*>(b_misc.as<char>() + 16);
  unsigned* absmax = reinterpret_cast<unsigned*>(b_misc.as<char>() + 32);

  // fixed-point scale from the largest |feature|
  SC_CUDA_TRY(cudaMemsetAsync(absmax, 0, sizeof(unsigned), s));
  absmax_bits_kernel<<<grid, kB, 0, s>>>(F, n * d, absmax);
  SC_CUDA_TRY(cudaGetLastError());
  unsigned amax_bits = 0;
  SC_CUDA_TRY(cudaMemcpyAsync(&amax_bits, absmax, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
  SC_CUDA_TRY(cudaStreamSynchronize(s));
  float amax;
  std::memcpy(&amax, &amax_bits, sizeof(float));
  if (!std::isfinite(amax)) return fail(SC_ERR_ARG, "features contain inf/nan");
  int E = 0;
  if (amax > 0.0f) { std::frexp((double)amax, &E); }   // amax < 2^E
  const int shift = 87 - E;

  // centroid tiles for smem (assign: kt*d doubles; accum: 3*kt*d + kt u64)
  const size_t smem_cap = 96 * 1024;
  int kt_assign = std::max(1, std::min(k, (int)(smem_cap / (sizeof(double) * d))));
  int kt_acc = std::max(1, std::min(k, (int)((smem_cap / sizeof(unsigned long long)) / (3 * (size_t)d + 1))));
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(assign_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_cap);
    cudaFuncSetAttribute(centroid_accum_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_cap);
    attr_set = true;
  }

  auto assign_all = [&](int32_t* out_lab, const int32_t* old, double* inertia, int* nchanged) -> int {
    SC_CUDA_TRY(cudaMemsetAsync(changed, 0, sizeof(int), s));
    for (int c0 = 0; c0 < k; c0 += kt_assign) {
      const int kt = std::min(kt_assign, k - c0);
      const int last = c0 + kt >= k;
      assign_kernel<<<grid, kB, sizeof(double) * kt * d, s>>>(F, n, d, C, c0, kt, c0 == 0, last, out_lab,
                                                               b_dmin.as<double>(), old, changed,
                                                               b_part.as<double>());
      SC_CUDA_TRY(cudaGetLastError());
    }
    std::vector<double> part(grid);
    int h_changed = 0;
    SC_CUDA_TRY(cudaMemcpyAsync(part.data(), b_part.as<double>(), sizeof(double) * grid, cudaMemcpyDeviceToHost, s));
    SC_CUDA_TRY(cudaMemcpyAsync(&h_changed, changed, sizeof(int), cudaMemcpyDeviceToHost, s));
    SC_CUDA_TRY(cudaStreamSynchronize(s));
    double tot = 0.0;
    for (double v : part) tot += v;
    *inertia = tot;
    *nchanged = h_changed;
    return SC_OK;
  };

  auto update = [&](const int32_t* cur) -> int {
    SC_CUDA_TRY(cudaMemsetAsync(b_limbs.ptr, 0, sizeof(unsigned long long) * 3 * k * d, s));
    SC_CUDA_TRY(cudaMemsetAsync(b_cnt.ptr, 0, sizeof(unsigned long long) * k, s));
    for (int c0 = 0; c0 < k; c0 += kt_acc) {
      const int kt = std::min(kt_acc, k - c0);
      const size_t sm = sizeof(unsigned long long) * (3 * (size_t)kt * d + kt);
      centroid_accum_kernel<<<grid, kB, sm, s>>>(F, cur, n, d, c0, kt, shift, b_limbs.as<unsigned long long>(), k,
                                                 b_cnt.as<unsigned long long>(), 1);
      SC_CUDA_TRY(cudaGetLastError());
    }
    centroid_finalize_kernel<<<std::max(1, std::min(grid, (k * d + kB - 1) / kB)), kB, 0, s>>>(
        b_limbs.as<unsigned long long>(), b_cnt.as<unsigned long long>(), k, d, shift, C);
    SC_CUDA_TRY(cudaGetLastError());
    return SC_OK;
  };

  double best_inertia = INFINITY;
  int best_r = -1, best_it = 0;
  std::vector<double> best_C((size_t)k * d);
  std::vector<double> u(k);
  std::vector<double> bsum(G), prefix(G + 1);
  for (int r = 0; r < restarts; ++r) {
    for (int t = 0; t < k; ++t)
      u[t] = uniforms_host ? uniforms_host[(size_t)r * k + t] : uniform_host(seed, 1, (uint64_t)r * k + t);
    // ---- k-means++ seeding
    int64_t idx = std::min<int64_t>((int64_t)std::floor(u[0] * n), n - 1);
    row_to_centroid_kernel<<<1, 128, 0, s>>>(F, idx, d, C);
    d2_update_kernel<<<grid, kB, sizeof(double) * d, s>>>(F, n, d, C, b_d2.as<double>(), 1);
    SC_CUDA_TRY(cudaGetLastError());
    for (int t = 1; t < k; ++t) {
      range_sums_kernel<<<G, kB, 0, s>>>(b_d2.as<double>(), n, chunk, b_part.as<double>());
      SC_CUDA_TRY(cudaMemcpyAsync(bsum.data(), b_part.as<double>(), sizeof(double) * G, cudaMemcpyDeviceToHost, s));
      SC_CUDA_TRY(cudaStreamSynchronize(s));
      prefix[0] = 0.0;
      for (int b = 0; b < G; ++b) prefix[b + 1] = prefix[b] + bsum[b];
      const double total = prefix[G];
      if (!(total > 0.0)) {
        idx = std::min<int64_t>((int64_t)std::floor(u[t] * n), n - 1);
      } else {
        const double target = u[t] * total;
        int b = 0;
        while (b < G - 1 && !(prefix[b + 1] > target)) ++b;
        const int64_t b0 = (int64_t)b * chunk, b1 = std::min<int64_t>(n, b0 + chunk);
        range_select_kernel<<<1, 32, 0, s>>>(b_d2.as<double>(), b0, b1, prefix[b], target, sel);
        SC_CUDA_TRY(cudaMemcpyAsync(&idx, sel, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        SC_CUDA_TRY(cudaStreamSynchronize(s));
      }
      row_to_centroid_kernel<<<1, 128, 0, s>>>(F, idx, d, C + (size_t)t * d);
      d2_update_kernel<<<grid, kB, sizeof(double) * d, s>>>(F, n, d, C + (size_t)t * d, b_d2.as<double>(), 0);
      SC_CUDA_TRY(cudaGetLastError());
    }
    // ---- Lloyd
    double inertia = 0.0;
    int nchg = 0;
    SC_TRY(assign_all(lab, nullptr, &inertia, &nchg));
    int it = 0;
    for (it = 1; it <= max_iter; ++it) {
      SC_TRY(update(lab));
      SC_TRY(assign_all(nw, lab, &inertia, &nchg));
      if (nchg == 0) break;
      std::swap(lab, nw);
    }
    if (it > max_iter) it = max_iter;
    if (inertia < best_inertia) {
      best_inertia = inertia;
      best_r = r;
      best_it = it;
      SC_CUDA_TRY(cudaMemcpyAsync(labels_dev, lab, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, s));
      SC_CUDA_TRY(cudaMemcpyAsync(best_C.data(), C, sizeof(double) * k * d, cudaMemcpyDeviceToHost, s));
      SC_CUDA_TRY(cudaStreamSynchronize(s));
    }
  }
  if (best_r < 0) return fail(SC_ERR_ARG, "k-means produced no finite inertia");
  if (centroids_host) std::memcpy(centroids_host, best_C.data(), sizeof(double) * k * d);
  if (inertia_out) *inertia_out = best_inertia;
  if (iters_out) *iters_out = best_it;
  if (best_out) *best_out = best_r;
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
