// k-means assignment screen on the 5th-generation tensor cores (tcgen05.mma kind::tf32,
// accumulators in TMEM).
//
// PAPER.md §2.2 step 4 (l.109-113), §4.1 step 6 (l.323-328): k-means on the feature rows
// with the Euclidean distance; the decisions follow DESIGN.md R8 (fp64, ascending-q sums,
// lowest index on ties).  Like the fp32 screen (assign_screen_kernel, sc_kmeans.cu), this
// pass only has to PROVE which centroid is the unique exact argmin of a point, with a
// rigorous error bound; the exact fp64 distance of the proven winner is then computed, and
// every point it cannot decide goes to the exact fp64 scan (assign3_kernel).  Labels are
// therefore bit-identical to a full fp64 scan whatever the tensor cores' rounding.
//
// Formulation.  A point x with current label a is screened in coordinates centred on c_a
// (the points are grouped by their current label, 128 per tile): y = fl32(x - fl32(c_a)),
// z_j = fl32(c_j - c_a), and ||x - c_j||^2 = ||y||^2 + ||z_j||^2 - 2 y.z_j up to the
// centring errors.  The tensor cores compute S_j = y.z_j for the tile's 128 points and all
// centroids in one M = 128 x N = k (rounded up to 8) x K = d (rounded up to 8) MMA chain
// (tf32 operands, fp32 accumulation in TMEM).  Centring keeps the products' magnitudes at
// ||y|| ||z_j|| (the point's distance to its own centroid times the centroid gaps) instead of
// ||x|| ||c_j||: the uncentred expanded form left 44 % of the configs[3] points undecided in
// fp32.
//
// Bound (all in fp64, u = 2^-24, eps_s = 2^-10 + 2^-22 + (K + 2) 2^-23 (1 + 2^-10): tf32
// rounding of both operands (cvt.rna: 2^-11 each) and a K-term fp32 accumulation in any order
// with at worst truncating adds):
//   |S_j - y.z_j|            <= eps_s ||y|| ||z_j||
//   delta_j (centring error) <= u (||y|| + ||c_a|| + ||z_j||) + 2^-51 C_m + tiny <= delta
//                               (delta: the same with max_j ||z_j||)
//   |D_j - rho_j^2|          <= 2 eps_s ||y|| ||z_j|| + 2 (||y|| + ||z_j|| + delta) delta
//                               + delta^2 + 2^-49 (Y2 + Z2_j + 2 |S_j|)  =: E_j
//   (the 2^-49 term covers the fp64 evaluation of D_j and E_j; every term is inflated by 1e-6)
// with D_j = Y2 + Z2_j - 2 S_j (Y2, Z2_j the fp64 squared norms of the fp32 vectors) and rho_j
// the exact distance of the fp32 point to the fp64 centroid.  The point is decided when
// min_{j != b} (D_j - E_j) > (D_b + E_b)(1 + 1e-12), b = argmin D_j (the 1e-12 covers the fp64
// evaluation of the winner's distance, as in the fp32 screen).  lo = sqrt of that minimum
// (times 1 - 1e-12) is a lower bound of the distance to every other centroid (Hamerly).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "sc_internal.cuh"

namespace sc {
namespace {

constexpr int kTM = 128;   // points per tile (TMEM lanes)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major, no swizzle: the 16-byte chunk (row r, k-chunk j) sits at
// ((r % 8) + (r / 8) * SBO + j * LBO) * 16 bytes; here LBO = 128 B, SBO = KC * 128 B
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;   // descriptor version (sm_100)
  return d;                  // base offset 0, lbo mode 0, SWIZZLE_NONE
}
__device__ __forceinline__ uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ float to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
// offset (in floats) of element (row r, column q) in the canonical K-major layout
__device__ __forceinline__ int canon(int r, int q, int KC) {
  return ((r & 7) + (r >> 3) * (8 * KC) + (q >> 2) * 8) * 4 + (q & 3);
}

struct TcArgs {
  const float* F;        // n x d
  const double* C;       // k x d (fp64 centroids)
  const float* Cf;       // k x d (fp32 copies)
  const double* cm;      // max_c ||c|| (rounded up)
  int n_items_max;
  const int* items;      // [item][2]: cluster, first position in gperm
  const int* n_items;    // device
  const int64_t* goff;   // [k + 1] cluster offsets in gperm
  const int32_t* gperm;  // points grouped by current label
  int k, d, Dp, NT, tmem_cols;
  int v4;                // rows and centroids 16-byte aligned (d % 4 == 0): vector staging
  int32_t* lab;
  double* dmin;
  double* lo;
  int32_t* amb;
  int* amb_len;
};

__global__ void __launch_bounds__(kTM) assign_tc_kernel(TcArgs a) {
  const int KC = a.Dp / 4;
  extern __shared__ __align__(1024) unsigned char tsm[];
  float* sA = reinterpret_cast<float*>(tsm);                    // [128][Dp] canonical
  float* sB = sA + (size_t)kTM * a.Dp;                          // [NT][Dp] canonical
  double* sZ2 = reinterpret_cast<double*>(sB + (size_t)a.NT * a.Dp);   // [NT]
  double* sZn = sZ2 + a.NT;                                     // [NT]
  double* sY2 = sZn + a.NT;                                     // [128]
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base;
  __shared__ double s_ca_norm, s_zmax;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(a.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  const int items = *a.n_items;
  const double u = 0x1p-24;
  const double eps_s = 0x1p-10 + 0x1p-22 + (a.Dp + 2) * 0x1p-23 * (1.0 + 0x1p-10);
  const double Cm = *a.cm;
  int cur = -1;   // cluster whose centred centroids sit in sB
  uint32_t phase = 0;
  // contiguous item ranges per CTA: consecutive items mostly share a cluster (centred
  // centroids staged once per cluster)
  const int per = (items + gridDim.x - 1) / gridDim.x;
  const int it0 = blockIdx.x * per, it1 = min(items, it0 + per);
  for (int it = it0; it < it1; ++it) {
    const int ca = a.items[2 * it], start = a.items[2 * it + 1];
    const int64_t cend = a.goff[ca + 1];
    const int cnt = (int)min((int64_t)kTM, cend - (a.goff[ca] + start));
    const int32_t* pts = a.gperm + a.goff[ca] + start;
    // ---- centred centroids z_j = fl32(c_j - c_a), their squared norms (once per cluster)
    if (ca != cur) {
      const double* cA = a.C + (size_t)ca * a.d;
      for (int e = tid; e < a.NT * a.Dp; e += kTM) {
        const int j = e / a.Dp, q = e % a.Dp;
        float z = 0.f;
        if (j < a.k && q < a.d) z = (float)(a.C[(size_t)j * a.d + q] - cA[q]);
        sB[canon(j, q, KC)] = z;   // rounded to tf32 below, after the norms
      }
      __syncthreads();
      for (int j = tid; j < a.NT; j += kTM) {
        double s2 = 0.0;
        for (int q = 0; q < a.Dp; ++q) {
          const double z = sB[canon(j, q, KC)];
          s2 += z * z;
        }
        sZ2[j] = s2;
        sZn[j] = sqrt(s2) * (1.0 + 1e-15);
      }
      if (tid == 0) {
        double s2 = 0.0;
        for (int q = 0; q < a.d; ++q) s2 += cA[q] * cA[q];
        s_ca_norm = sqrt(s2) * (1.0 + 1e-15);
      }
      __syncthreads();
      if (tid == 0) {
        double zm = 0.0;
        for (int j = 0; j < a.NT; ++j) zm = fmax(zm, sZn[j]);
        s_zmax = zm;
      }
      for (int e = tid; e < a.NT * a.Dp; e += kTM) {
        const int j = e / a.Dp, q = e % a.Dp;
        float* p = sB + canon(j, q, KC);
        *p = to_tf32(*p);
      }
      cur = ca;
    }
    // ---- centred points y = fl32(x - fl32(c_a)), tf32 copies for the MMA, fp64 ||y||^2
    // (a warp takes a row, lanes along it)
    const float* cAf = a.Cf + (size_t)ca * a.d;
    if (a.v4) {
      // thread tid stages its own point (row tid = TMEM lane tid of the epilogue): its row's
      // 16-byte chunks, up to 16 loads in flight, written to the canonical layout (the lanes
      // of a warp fill four contiguous 128-byte runs: no bank conflicts)
      const int r = tid;
      const int64_t gi = r < cnt ? pts[r] : -1;
      const float4* xr = reinterpret_cast<const float4*>(a.F + (gi >= 0 ? gi : 0) * a.d);
      const int nval = a.d / 4;
      double s2 = 0.0;
      for (int j0 = 0; j0 < KC; j0 += 16) {
        float4 xv[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) {
          const int j = j0 + t;
          xv[t] = (gi >= 0 && j < nval) ? __ldg(xr + j) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int t = 0; t < 16; ++t) {
          const int j = j0 + t;
          if (j >= KC) break;
          float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
          if (gi >= 0 && j < nval) {
            const float4 c = *reinterpret_cast<const float4*>(cAf + 4 * j);
            y = make_float4(__fsub_rn(xv[t].x, c.x), __fsub_rn(xv[t].y, c.y), __fsub_rn(xv[t].z, c.z),
                            __fsub_rn(xv[t].w, c.w));
          }
          s2 += (double)y.x * y.x + (double)y.y * y.y + (double)y.z * y.z + (double)y.w * y.w;
          *reinterpret_cast<float4*>(sA + ((r & 7) + (r >> 3) * (8 * KC) + j * 8) * 4) =
              make_float4(to_tf32(y.x), to_tf32(y.y), to_tf32(y.z), to_tf32(y.w));
        }
      }
      sY2[r] = s2;
    } else {
      for (int r = warp; r < kTM; r += 4) {
        double s2 = 0.0;
        const int64_t gi = r < cnt ? pts[r] : -1;
        for (int q = lane; q < a.Dp; q += 32) {
          float y = 0.f;
          if (gi >= 0 && q < a.d) y = __fsub_rn(a.F[gi * a.d + q], cAf[q]);
          s2 += (double)y * (double)y;
          sA[canon(r, q, KC)] = to_tf32(y);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
        if (lane == 0) sY2[r] = s2;
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // smem writes -> tensor core
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (tid == 0) {
      const uint32_t id = idesc_tf32(kTM, a.NT);
      for (int ks = 0; ks < a.Dp / 8; ++ks) {   // one MMA per 8 tf32 of K (two 16-byte chunks)
        const uint64_t da = umma_desc(smem_u32(sA) + ks * 256, 128, KC * 128);
        const uint64_t db = umma_desc(smem_u32(sB) + ks * 256, 128, KC * 128);
        const uint32_t acc = ks > 0;
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
            "l"(da), "l"(db), "r"(id), "r"(acc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(&bar))
                   : "memory");
    }
    asm volatile(
        "{\n.reg .pred P1;\nTCW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra TCW_%=;\n}\n" ::"r"(
            smem_u32(&bar)),
        "r"(phase)
        : "memory");
    phase ^= 1u;
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // ---- epilogue: thread tid owns point tid (TMEM lane tid)
    const double Y2 = sY2[tid];
    const double yn = sqrt(Y2) * (1.0 + 1e-15);
    // E_j <= Ea zn_j + Eb0 + 2^-49 Z2_j + 2^-48 |S_j| with the centring error bounded by its
    // largest value over j (zmax = max_j ||z_j||): fewer fp64 operations per column
    const double dmx = u * (yn + s_ca_norm + s_zmax) + 0x1p-51 * Cm + 0x1p-120;
    const double Ea = (2.0 * eps_s * yn + 2.0 * dmx) * (1.0 + 1e-6);
    const double Eb0 = (2.0 * (yn + dmx) * dmx + dmx * dmx + 0x1p-49 * Y2 + 0x1p-100) * (1.0 + 1e-6);
    double Db = INFINITY, Eb = 0.0, m2 = INFINITY;
    int b = -1;
    for (int c0 = 0; c0 < a.NT; c0 += 8) {
      uint32_t v[8];
      const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                   : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int j = c0 + q;
        if (j >= a.k) break;
        const double S = (double)__uint_as_float(v[q]);
        const double Z2 = sZ2[j];
        const double D = Y2 + Z2 - 2.0 * S;
        const double E = fma(Ea, sZn[j], Eb0) + 0x1p-49 * (1.0 + 1e-6) * Z2 + 0x1p-48 * (1.0 + 1e-6) * fabs(S);
        if (D < Db) {
          if (b >= 0) m2 = fmin(m2, Db - Eb);
          b = j;
          Db = D;
          Eb = E;
        } else {
          m2 = fmin(m2, D - E);
        }
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    if (tid < cnt) {
      const int64_t gi = pts[tid];
      const double up = (Db + Eb) * (1.0 + 1e-12);
      const double low = (a.k == 1) ? (double)INFINITY : m2 * (1.0 - 1e-12);
      if (b >= 0 && low > up) {
        // proven unique argmin: its exact distance with the scan's arithmetic (R8)
        const double* c = a.C + (size_t)b * a.d;
        const float* x = a.F + gi * a.d;
        double acc = 0.0;
        for (int q = 0; q < a.d; ++q) {
          const double diff = __dsub_rn((double)__ldg(x + q), c[q]);
          acc = __dadd_rn(acc, __dmul_rn(diff, diff));
        }
        a.lab[gi] = b;
        a.dmin[gi] = acc;
        a.lo[gi] = isinf(low) ? (double)INFINITY : sqrt(fmax(low, 0.0));
      } else {
        a.amb[atomicAdd(a.amb_len, 1)] = static_cast<int32_t>(gi);
      }
    }
    __syncthreads();   // sA / TMEM reused by the next tile
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(a.tmem_cols));
}

// ---- grouping of the points to screen by their current label (counting sort).  Shared-
// memory histograms per block, one global atomic per (block, cluster): with k ~ 100 clusters,
// per-point global atomics on k counters serialise (measured ~1.7 ms per assignment at n = 10^6).
constexpr int kGChunk = 4096;   // points per block of the grouping kernels
__global__ void __launch_bounds__(256) group_hist_kernel(const int32_t* __restrict__ old_lab,
                                                         const int32_t* __restrict__ list,
                                                         const int* __restrict__ list_len, int64_t n, int k,
                                                         unsigned* __restrict__ cnt) {
  extern __shared__ unsigned sh_cnt[];
  const int64_t m = list ? (int64_t)*list_len : n;
  const int64_t b0 = (int64_t)blockIdx.x * kGChunk;
  if (b0 >= m) return;
  for (int c = threadIdx.x; c < k; c += blockDim.x) sh_cnt[c] = 0u;
  __syncthreads();
  const int64_t b1 = min(m, b0 + kGChunk);
  for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) atomicAdd(&sh_cnt[old_lab[list ? list[i] : i]], 1u);
  __syncthreads();
  for (int c = threadIdx.x; c < k; c += blockDim.x)
    if (sh_cnt[c]) atomicAdd(&cnt[c], sh_cnt[c]);
}

// offsets (exclusive scan of the counts), work items (cluster, first position) of <= 128
// points, cursors zeroed; one block
__global__ void __launch_bounds__(256) group_plan_kernel(const unsigned* __restrict__ cnt, int k,
                                                         int64_t* __restrict__ off, unsigned* __restrict__ cursor,
                                                         int* __restrict__ items, int* __restrict__ n_items) {
  __shared__ long long s_c[256];
  __shared__ int s_i[256];
  __shared__ long long carry;
  __shared__ int carry_i;
  const int tid = threadIdx.x;
  if (tid == 0) { carry = 0; carry_i = 0; }
  __syncthreads();
  for (int base = 0; base < k; base += 256) {
    const int c = base + tid;
    const long long cc = c < k ? (long long)cnt[c] : 0;
    const int ni = (int)((cc + kTM - 1) / kTM);
    s_c[tid] = cc;
    s_i[tid] = ni;
    __syncthreads();
    for (int o = 1; o < 256; o <<= 1) {
      const long long x = tid >= o ? s_c[tid - o] : 0;
      const int y = tid >= o ? s_i[tid - o] : 0;
      __syncthreads();
      s_c[tid] += x;
      s_i[tid] += y;
      __syncthreads();
    }
    if (c < k) {
      off[c] = carry + s_c[tid] - cc;
      cursor[c] = 0u;
      const int i0 = carry_i + s_i[tid] - ni;
      for (int t = 0; t < ni; ++t) {
        items[2 * (i0 + t)] = c;
        items[2 * (i0 + t) + 1] = t * kTM;
      }
    }
    __syncthreads();
    if (tid == 255) { carry += s_c[255]; carry_i += s_i[255]; }
    __syncthreads();
  }
  if (tid == 0) {
    off[k] = carry;
    *n_items = carry_i;
  }
}

__global__ void __launch_bounds__(256) group_scatter_kernel(const int32_t* __restrict__ old_lab,
                                                            const int32_t* __restrict__ list,
                                                            const int* __restrict__ list_len, int64_t n, int k,
                                                            const int64_t* __restrict__ off,
                                                            unsigned* __restrict__ cursor,
                                                            int32_t* __restrict__ gperm) {
  extern __shared__ unsigned sh_sc[];   // [k] block counts, [k] block bases, [k] ranks
  unsigned* bcnt = sh_sc;
  unsigned* bbase = sh_sc + k;
  unsigned* brank = sh_sc + 2 * k;
  const int64_t m = list ? (int64_t)*list_len : n;
  const int64_t b0 = (int64_t)blockIdx.x * kGChunk;
  if (b0 >= m) return;
  for (int c = threadIdx.x; c < k; c += blockDim.x) { bcnt[c] = 0u; brank[c] = 0u; }
  __syncthreads();
  const int64_t b1 = min(m, b0 + kGChunk);
  for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) atomicAdd(&bcnt[old_lab[list ? list[i] : i]], 1u);
  __syncthreads();
  for (int c = threadIdx.x; c < k; c += blockDim.x) bbase[c] = bcnt[c] ? atomicAdd(&cursor[c], bcnt[c]) : 0u;
  __syncthreads();
  for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
    const int64_t p = list ? list[i] : i;
    const int c = old_lab[p];
    gperm[off[c] + bbase[c] + atomicAdd(&brank[c], 1u)] = static_cast<int32_t>(p);
  }
}

}  // namespace

bool tc_screen_supported(int k, int d) {
  const char* e = std::getenv("SC_KMEANS_TC");
  if (e && std::atoi(e) == 0) return false;
  const int NT = (k + 7) / 8 * 8, Dp = (d + 7) / 8 * 8;
  const size_t smem = (size_t)(kTM + NT) * Dp * 4 + (size_t)(2 * NT + kTM) * 8;
  return k >= 2 && NT <= 256 && smem <= 200 * 1024;
}

int tc_screen(const float* F, int64_t n, int d, const double* C, const float* Cf, const double* cm, int k,
              const int32_t* old_lab, const int32_t* list, const int* list_len, int32_t* lab, double* dmin,
              double* lo, int32_t* amb, int* amb_len, TcWork& w, cudaStream_t s) {
  const int NT = (k + 7) / 8 * 8, Dp = (d + 7) / 8 * 8;
  const int max_items = (int)((n + kTM - 1) / kTM) + k;
  SC_TRY(w.cnt.ensure(sizeof(unsigned) * 2 * (size_t)k, s));
  SC_TRY(w.off.ensure(sizeof(int64_t) * (size_t)(k + 1), s));
  SC_TRY(w.items.ensure(sizeof(int) * (2 * (size_t)max_items + 1), s));
  SC_TRY(w.gperm.ensure(sizeof(int32_t) * (size_t)std::max<int64_t>(1, n), s));
  unsigned* cnt = w.cnt.as<unsigned>();
  unsigned* cursor = cnt + k;
  int* n_items = w.items.as<int>() + 2 * (size_t)max_items;
  int sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  SC_CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(unsigned) * k, s));
  const int pgrid = (int)std::max<int64_t>(1, (n + kGChunk - 1) / kGChunk);   // (list: <= n entries)
  group_hist_kernel<<<pgrid, 256, sizeof(unsigned) * k, s>>>(old_lab, list, list_len, n, k, cnt);
  group_plan_kernel<<<1, 256, 0, s>>>(cnt, k, w.off.as<int64_t>(), cursor, w.items.as<int>(), n_items);
  group_scatter_kernel<<<pgrid, 256, sizeof(unsigned) * 3 * k, s>>>(old_lab, list, list_len, n, k,
                                                                    w.off.as<int64_t>(), cursor,
                                                                    w.gperm.as<int32_t>());
  SC_CUDA_TRY(cudaGetLastError());
  TcArgs a{};
  a.F = F;
  a.C = C;
  a.Cf = Cf;
  a.cm = cm;
  a.n_items_max = max_items;
  a.items = w.items.as<int>();
  a.n_items = n_items;
  a.goff = w.off.as<int64_t>();
  a.gperm = w.gperm.as<int32_t>();
  a.k = k;
  a.d = d;
  a.Dp = Dp;
  a.NT = NT;
  a.tmem_cols = NT <= 32 ? 32 : NT <= 64 ? 64 : NT <= 128 ? 128 : 256;
  a.v4 = (d % 4 == 0) && ((uintptr_t)F % 16 == 0) && ((uintptr_t)Cf % 16 == 0);
  a.lab = lab;
  a.dmin = dmin;
  a.lo = lo;
  a.amb = amb;
  a.amb_len = amb_len;
  const int smem = (int)((size_t)(kTM + NT) * Dp * 4 + (size_t)(2 * NT + kTM) * 8);
  static int attr = 0;
  if (smem > attr) {
    SC_CUDA_TRY(cudaFuncSetAttribute(assign_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr = 200 * 1024;
  }
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, assign_tc_kernel, kTM, smem);
  occ = std::max(1, std::min(occ, 512 / a.tmem_cols));   // TMEM: 512 columns per SM
  const int grid = (int)std::min<int64_t>(max_items, (int64_t)sms * occ);
  assign_tc_kernel<<<grid, kTM, smem, s>>>(a);
  SC_CUDA_TRY(cudaGetLastError());
  return SC_OK;
}

}  // namespace sc
