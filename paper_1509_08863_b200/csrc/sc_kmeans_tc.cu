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
// Bound (u = 2^-24, eps_s = 2^-10 + 2^-22 + (K + 2) 2^-23 (1 + 2^-10): tf32 rounding of both
// operands (cvt.rna: 2^-11 each) and a K-term fp32 accumulation in any order with at worst
// truncating adds):
//   |S_j - y.z_j|            <= eps_s ||y|| ||z_j||
//   delta_j (centring error) <= u (||y|| + ||c_a|| + ||z_j||) + 2^-51 C_m + tiny <= delta
//                               (delta: the same with max_j ||z_j||)
//   |D*_j - rho_j^2|         <= 2 eps_s ||y|| ||z_j|| + 2 (||y|| + ||z_j|| + delta) delta + delta^2
//                             = Ea ||z_j|| + Eb0 =: E_j
// with D*_j = Y2 + Z2_j - 2 S_j exactly (Y2, Z2_j the exact squared norms of the fp32
// vectors) and rho_j the exact distance of the fp32 point to the fp64 centroid.  Z2_j is an
// fp64 sum (rounding ~2^-47 relative, inside kappa below); Y2 is summed in fp32 and enclosed
// in [Y2c (1 - gamma), Y2c (1 + gamma)], gamma = (K + 2) 2^-24: the lower end enters the lower
// bounds L_j (V below), the upper end the winner's upper bound U and ||y||.  Ea, Eb0 are per point (fp64, inflated by 1e-6; Ea rounded up to fp32).
// Per column the epilogue evaluates in fp32, with kappa = 2^-20,
//   L_j = fma(-2 kappa, |S_j|, fma(-2, S_j, fma(-Ea, zn_j, W_j) + V)),
//   W_j = fl32(fl32(Z2_j)(1 - kappa)),  zn_j >= ||z_j||,  V = fl32_down(Y2l (1 - kappa) - Eb0),
// i.e. D*_j - E_j - kappa M_j (M_j = Y2 + Z2_j + 2 |S_j|) up to seven roundings of at most
// 2^-24 M_j each (< 2^-21 M_j < kappa M_j), so L_j <= rho_j^2 rigorously.  With b = argmin_j L_j
// and U = D*_b + E_b evaluated in fp64 from S_b (an upper bound of rho_b^2), the point is
// decided when min_{j != b} L_j (1 - 1e-12) > U (1 + 1e-12): rho_b^2 is then below every other
// rho_j^2 by a relative gap far larger than the fp64 evaluation of the distances in R8, so the
// fp64 scan picks b too.  lo = sqrt of the left-hand side is a lower bound of the distance to
// every other centroid (Hamerly).  Points with ||y||^2 or a ||z_j||^2 >= 1e30 (fp32 overflow)
// are left undecided.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <utility>
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
  const int* ioff;       // [k + 1] exclusive prefix of the clusters' tile counts (<= 128 points)
  const int* n_items;    // device
  const int64_t* goff;   // [k + 1] cluster offsets in gperm
  const int32_t* gperm;  // points grouped by current label
  int k, d, Dp, NT, tmem_cols;
  int tmem_tile;         // TMEM columns per 128-point tile (the second tile's accumulator offset)
  int v4;                // rows and centroids 16-byte aligned (d % 4 == 0): vector staging
  const float* panels;   // [k][panel_floats]: per current cluster a, see tc_panel_kernel
  const double* pscal;   // [k][16]: see tc_panel_kernel
  int panel_floats;      // NT * Dp + 3 * NT
  int* ctr;              // item-chunk counter (zeroed by group_plan_kernel)
  unsigned long long* prof;   // env SC_TC_PROFILE (tooling): per-phase clock64 sums of thread 0
  int32_t* fix;          // decided points whose exact distance tc_fix_kernel computes
  int* fix_len;
  int32_t* lab;
  double* dmin;
  double* lo;
  int32_t* amb;
  int* amb_len;
};

// prefetched 16-byte chunks per point: 16 (d <= 64, 3 CTAs per SM) or 32 (d <= 128, the
// one-CTA-per-SM instantiation large k x d needs: registers are not the limit there)
constexpr int kPV = 16;
constexpr int kPVWide = 32;
constexpr double kKappa = 0x1p-20;   // fp32 evaluation budget of the per-column bound (above)
constexpr float kKappaF = 0x1p-20f;
constexpr int kChunk = 4; // items a CTA takes per counter increment

// shared-memory bytes of assign_tc_kernel
// (TP points per CTA: one or two 128-point MMA tiles sharing the cluster's panel)
__host__ __device__ inline size_t tc_smem_bytes(int NT, int Dp, int TP = kTM) {
  return (size_t)(TP + NT) * Dp * 4 + (size_t)(3 * NT + Dp) * 4 + (size_t)(TP + Dp) * 8;
}

// Per-cluster panels, once per assignment (grid k x NT/32, a warp per 4 centroids): for the
// current cluster a, the centred centroids z_j = fl32(c_j - c_a) rounded to tf32 in the MMA's
// canonical K-major layout, then per column {W_j = fl32(fl32(||z_j||^2) (1 - kappa)), ||z_j||
// rounded up to fp32}, then fl32(||z_j||^2); padding columns j >= k get W_j = +inf (never a
// candidate).  The squared norms are fp64 sums of the fp32 (not yet tf32-rounded) z_j.
// pscal[16 a]: ||c_a|| (1 + 1e-9); pscal[16 a + 1 + jb]: max ||z_j|| (fp64, times 1 + 1e-15)
// over the block's 32 columns, +inf when a ||z_j||^2 overflows fp32.
__global__ void __launch_bounds__(256) tc_panel_kernel(const double* __restrict__ C, int k, int d, int Dp, int NT,
                                                       float* __restrict__ panels, double* __restrict__ pscal,
                                                       int panel_floats) {
  __shared__ double s_zn[32];
  const int a = blockIdx.x, jb = blockIdx.y, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int KC = Dp / 4;
  const double* cA = C + (size_t)a * d;
  float* P = panels + (size_t)a * panel_floats;
#pragma unroll 1
  for (int r = 0; r < 4; ++r) {
    const int jl = warp * 4 + r, j = jb * 32 + jl;
    if (j >= NT) {   // (NT: k rounded up to 16; the last block may be half empty)
      if (lane == 0) s_zn[jl] = 0.0;
      continue;
    }
    double s2 = 0.0;
    for (int q = lane; q < Dp; q += 32) {
      float z = 0.f;
      if (j < k && q < d) z = (float)(C[(size_t)j * d + q] - cA[q]);
      s2 += (double)z * (double)z;
      P[canon(j, q, KC)] = to_tf32(z);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    if (lane == 0) {
      const double zn = sqrt(s2) * (1.0 + 1e-15);
      const float z2f = (float)s2;
      const bool pad = j >= k;
      P[NT * Dp + 2 * j] = pad ? INFINITY : __fmul_rn(z2f, 1.f - kKappaF);   // W_j
      P[NT * Dp + 2 * j + 1] = pad ? 0.f : __double2float_ru(zn);
      P[NT * Dp + 2 * NT + j] = z2f;
      s_zn[jl] = (!pad && !(z2f < 1e30f)) ? (double)INFINITY : zn;
    }
  }
  __syncthreads();
  if (warp == 0) {
    double zm = s_zn[lane], s2 = 0.0;
    if (jb == 0)
      for (int q = lane; q < d; q += 32) s2 += cA[q] * cA[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      zm = fmax(zm, __shfl_xor_sync(0xffffffffu, zm, o));
      s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    }
    if (lane == 0) {
      pscal[16 * (size_t)a + 1 + jb] = zm;
      if (jb == 0) pscal[16 * (size_t)a] = sqrt(s2) * (1.0 + 1e-9);
    }
  }
}

// per-thread state of the epilogue's column scan: smallest / second smallest L and the
// smallest's S and index, for even and odd columns separately
struct ColTrack {
  float L1e = INFINITY, L2e = INFINITY, Sbe = 0.f, L1o = INFINITY, L2o = INFINITY, Sbo = 0.f;
  int be = -1, bo = -1;
};

// NW accumulator columns c0 .. c0 + NW - 1 of this thread's TMEM lane: L_j (bound in the file
// header) and the tracking update
template <int NW>
__device__ __forceinline__ void tc_columns(uint32_t taddr, int c0, const float4* __restrict__ sWZ2, float Eaf,
                                           float V, ColTrack& t) {
  uint32_t v[NW];
  if constexpr (NW == 32) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
  } else {
    static_assert(NW == 16, "32- or 16-column loads");
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
  }
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int q = 0; q < NW; q += 2) {
    const float4 wz = sWZ2[(c0 + q) >> 1];   // {W_j, zn_j, W_j+1, zn_j+1}
    const float S0 = __uint_as_float(v[q]), S1 = __uint_as_float(v[q + 1]);
    const float L0 = fmaf(-2.f * kKappaF, fabsf(S0), fmaf(-2.f, S0, fmaf(-Eaf, wz.y, wz.x) + V));
    const float Lx = fmaf(-2.f * kKappaF, fabsf(S1), fmaf(-2.f, S1, fmaf(-Eaf, wz.w, wz.z) + V));
    t.L2e = fminf(t.L2e, fmaxf(t.L1e, L0));
    const bool lte = L0 < t.L1e;
    t.L1e = fminf(t.L1e, L0);
    t.Sbe = lte ? S0 : t.Sbe;
    t.be = lte ? c0 + q : t.be;
    t.L2o = fminf(t.L2o, fmaxf(t.L1o, Lx));
    const bool lto = Lx < t.L1o;
    t.L1o = fminf(t.L1o, Lx);
    t.Sbo = lto ? S1 : t.Sbo;
    t.bo = lto ? c0 + q + 1 : t.bo;
  }
}

// TP = 128: one MMA tile per CTA.  TP = 256 (large k x d, where shared memory allows one CTA per
// SM): two 128-point tiles of the same cluster per CTA, both multiplied by the one staged panel
// into two TMEM accumulators (columns [0, tmem_tile) and [tmem_tile, 2 tmem_tile)); warps w and
// w + 4 read the same TMEM lanes (w % 4) of their own accumulator -- 8 warps per SM instead of 4.
template <int PV, int MINB, int TP>
__global__ void __launch_bounds__(TP, MINB) assign_tc_kernel(TcArgs a) {
  const int KC = a.Dp / 4;
  extern __shared__ __align__(1024) unsigned char tsm[];
  float* sA = reinterpret_cast<float*>(tsm);                    // [128][Dp] canonical
  float* sB = sA + (size_t)TP * a.Dp;                           // [NT][Dp] canonical, then:
  const float2* sWZ = reinterpret_cast<const float2*>(sB + (size_t)a.NT * a.Dp);   // [NT] {W_j, zn_j}
  const float* sZ2f = sB + (size_t)a.NT * a.Dp + 2 * a.NT;      // [NT] fl32(||z_j||^2)
  float* s_caf = sB + (size_t)a.NT * a.Dp + 3 * a.NT;           // [Dp] fl32(c_a)
  double* sY2 = reinterpret_cast<double*>(s_caf + a.Dp);        // [128]
  double* s_ca = sY2 + TP;                                      // [Dp]: c_a (fp64)
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base;
  __shared__ double s_ca_norm, s_zmax;
  __shared__ int s_zbad, s_chunk;
  __shared__ int s_ioff[257];
  __shared__ long long s_goff[257];
  __shared__ long long s_nidx[TP];   // point of each row of the tile whose rows are copied next
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
  for (int c = tid; c <= a.k; c += TP) {
    s_ioff[c] = a.ioff[c];
    s_goff[c] = a.goff[c];
  }
  __syncthreads();
  // tile i -> (cluster, first position): the last cluster whose prefix is <= i
  auto tile_of = [&](int i, int& ca, int& start) {
    int lo = 0, hi = a.k - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_ioff[mid] <= i) lo = mid; else hi = mid - 1;
    }
    ca = lo;
    start = (i - s_ioff[lo]) * TP;
  };
  const double u = 0x1p-24;
  const double eps_s = 0x1p-10 + 0x1p-22 + (a.Dp + 2) * 0x1p-23 * (1.0 + 0x1p-10);
  const double Cm = *a.cm;
  const int nval = a.d / 4;
  // d <= 64 with 16-byte rows: the next tile's rows are loaded into registers while the
  // tensor cores and the epilogue work on the current one
  const bool pref = a.v4 && nval <= PV;
  int cur = -1;   // cluster whose panel sits in sB
  uint32_t phase = 0;
  // dynamic schedule: chunks of kChunk consecutive tiles (consecutive tiles mostly share a
  // cluster, so the panel is staged about once per chunk or less).  Two tiles ahead are
  // known: the next tile's rows are loaded during this tile's MMA and epilogue from an index
  // loaded one tile earlier (no dependent global load on the critical path).
  if (tid == 0) s_chunk = atomicAdd(a.ctr, kChunk);
  __syncthreads();
  int it = s_chunk, ca = 0, start = 0;   // the current tile
  const int chunk_end0 = min(items, it + kChunk);
  if (it < items) tile_of(it, ca, start);
  // the successor of a tile inside its chunk: the next tile of the same cluster or the first of
  // the next non-empty cluster
  auto walk = [&](int c, int st, int& c_n, int& st_n) {
    c_n = c;
    st_n = st + TP;
    if (st_n >= (s_ioff[c + 1] - s_ioff[c]) * TP) {
      c_n = c + 1;
      while (s_ioff[c_n + 1] == s_ioff[c_n]) ++c_n;
      st_n = 0;
    }
  };
  int it1 = items, ca1 = 0, st1 = 0, chunk_end1 = chunk_end0;   // the next tile
  if (it < items) {
    if (it + 1 < chunk_end0) {
      it1 = it + 1;
      walk(ca, start, ca1, st1);
    } else {
      __syncthreads();   // (all threads: the condition is uniform)
      if (tid == 0) s_chunk = atomicAdd(a.ctr, kChunk);
      __syncthreads();
      it1 = s_chunk;
      chunk_end1 = min(items, it1 + kChunk);
      if (it1 < items) tile_of(it1, ca1, st1);
    }
  }
  auto load_idx = [&](int c, int st) -> int64_t {
    const int64_t g0 = s_goff[c] + st;
    const int cnt = (int)min((int64_t)TP, (int64_t)(s_goff[c + 1] - g0));
    return tid < cnt ? (int64_t)a.gperm[g0 + tid] : (int64_t)-1;
  };
  // the next tile's raw rows are copied into sA, at their canonical positions, while the
  // epilogue of the current tile runs (sA is free once its MMA completed); a warp copies G rows
  // per instruction, lane = 16-byte chunk, so the loads are coalesced along each row (with one
  // row per thread they touched 32 lines per instruction).  Chunks past the row (padding to
  // Dp) and rows past the tile are zero-filled (src-size 0).
  const int G = KC <= 16 ? 2 : 1, LPR = 32 / G;
  auto copy_rows = [&]() {
    const int j = lane % LPR;
    for (int r = warp * G + lane / LPR; r < TP; r += (TP / 32) * G) {
      const int64_t gi = s_nidx[r];
      if (j < KC) {
        const bool ok = gi >= 0 && j < nval;
        const float* src = a.F + (ok ? gi * a.d + 4 * j : 0);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(sA + canon(r, 4 * j, KC))),
                     "l"(src), "r"(ok ? 16 : 0)
                     : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  int64_t gi_cur = -1, gi1 = -1;
  if (it < items) gi_cur = load_idx(ca, start);
  if (it1 < items) gi1 = load_idx(ca1, st1);
  if (pref && it < items) {
    s_nidx[tid] = gi_cur;
    __syncthreads();
    copy_rows();
  }
  unsigned long long pt[7] = {0, 0, 0, 0, 0, 0, 0};
  long long tprev = clock64();
  auto mark = [&](int i) {
    if (a.prof && tid == 0) {
      const long long t = clock64();
      pt[i] += (unsigned long long)(t - tprev);
      tprev = t;
    }
  };
  while (it < items) {
    mark(6);
    const int64_t g0 = s_goff[ca] + start;
    const int cnt = (int)min((int64_t)TP, (int64_t)(s_goff[ca + 1] - g0));
    const int32_t* pts = a.gperm + g0;
    // ---- the cluster's panel (tc_panel_kernel), c_a in fp64 and fp32
    if (ca != cur) {
      const float* P = a.panels + (size_t)ca * a.panel_floats;
      for (int e = tid; e < a.panel_floats / 4; e += TP)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sB + 4 * e)), "l"(P + 4 * e)
                     : "memory");
      asm volatile("cp.async.commit_group;" ::: "memory");
      for (int q = tid; q < a.Dp; q += TP) {
        s_ca[q] = q < a.d ? a.C[(size_t)ca * a.d + q] : 0.0;
        s_caf[q] = q < a.d ? a.Cf[(size_t)ca * a.d + q] : 0.f;
      }
      if (tid == 0) {
        const double* ps = a.pscal + 16 * (size_t)ca;
        double zm = 0.0;
        for (int jb = 0; jb < (a.NT + 31) / 32; ++jb) zm = fmax(zm, ps[1 + jb]);
        s_ca_norm = ps[0];
        s_zmax = zm;
        s_zbad = isinf(zm);
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
      __syncthreads();
      cur = ca;
    }
    if (pref) {   // this tile's raw rows (copy_rows) have landed in sA
      asm volatile("cp.async.wait_all;" ::: "memory");
      __syncthreads();
    }
    // the tile after next: the next of its chunk, else the first of a new chunk (taken before
    // the barrier below, read after it)
    const bool need_grab = it1 < items && it1 + 1 >= chunk_end1;
    if (need_grab && tid == 0) s_chunk = atomicAdd(a.ctr, kChunk);
    mark(0);
    // ---- centred points y = fl32(x - fl32(c_a)), tf32 copies for the MMA, fp64 ||y||^2; with
    // the prefetched rows also the exact (R8) distance to c_a, the usual winner
    double acc_a = 0.0;
    if (pref) {
      const int r = tid;
      float s2 = 0.f;   // ||y||^2 in fp32, sequential: within (K + 2) 2^-24 relative (epilogue)
#pragma unroll
      for (int t = 0; t < PV; ++t) {
        if (t >= KC) break;
        float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
        float4* slot = reinterpret_cast<float4*>(sA + ((r & 7) + (r >> 3) * (8 * KC) + t * 8) * 4);
        if (t < nval) {
          const float4 x = *slot;   // raw row (copy_rows), replaced in place by tf32(y) below
          const float4 c = *reinterpret_cast<const float4*>(s_caf + 4 * t);
          y = make_float4(__fsub_rn(x.x, c.x), __fsub_rn(x.y, c.y), __fsub_rn(x.z, c.z), __fsub_rn(x.w, c.w));
          const float xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const double diff = __dsub_rn((double)xs[e], s_ca[4 * t + e]);
            acc_a = __dadd_rn(acc_a, __dmul_rn(diff, diff));
          }
        }
        s2 = fmaf(y.w, y.w, fmaf(y.z, y.z, fmaf(y.y, y.y, fmaf(y.x, y.x, s2))));
        *slot = make_float4(to_tf32(y.x), to_tf32(y.y), to_tf32(y.z), to_tf32(y.w));
      }
      sY2[r] = (double)s2;
    } else if (a.v4) {
      const int r = tid;
      const int64_t gi = r < cnt ? pts[r] : -1;
      const float4* xr = reinterpret_cast<const float4*>(a.F + (gi >= 0 ? gi : 0) * a.d);
      double s2 = 0.0;
      for (int j0 = 0; j0 < KC; j0 += 16) {
        float4 xw[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) {
          const int j = j0 + t;
          xw[t] = (gi >= 0 && j < nval) ? __ldg(xr + j) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int t = 0; t < 16; ++t) {
          const int j = j0 + t;
          if (j >= KC) break;
          float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
          if (gi >= 0 && j < nval) {
            const float4 c = *reinterpret_cast<const float4*>(s_caf + 4 * j);
            y = make_float4(__fsub_rn(xw[t].x, c.x), __fsub_rn(xw[t].y, c.y), __fsub_rn(xw[t].z, c.z),
                            __fsub_rn(xw[t].w, c.w));
          }
          s2 += (double)y.x * y.x + (double)y.y * y.y + (double)y.z * y.z + (double)y.w * y.w;
          *reinterpret_cast<float4*>(sA + ((r & 7) + (r >> 3) * (8 * KC) + j * 8) * 4) =
              make_float4(to_tf32(y.x), to_tf32(y.y), to_tf32(y.z), to_tf32(y.w));
        }
      }
      sY2[r] = s2;
    } else {
      for (int r = warp; r < TP; r += TP / 32) {
        double s2 = 0.0;
        const int64_t gi = r < cnt ? pts[r] : -1;
        for (int q = lane; q < a.Dp; q += 32) {
          float y = 0.f;
          if (gi >= 0 && q < a.d) y = __fsub_rn(a.F[gi * a.d + q], s_caf[q]);
          s2 += (double)y * (double)y;
          sA[canon(r, q, KC)] = to_tf32(y);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
        if (lane == 0) sY2[r] = s2;
      }
    }
    mark(1);
    if (pref) s_nidx[tid] = gi1;   // rows copied after this tile's MMA (read after the barrier)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // smem writes -> tensor core
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    int it2 = items, ca2 = 0, st2 = 0, chunk_end2 = chunk_end1;
    if (it1 < items) {
      if (need_grab) {
        it2 = s_chunk;
        chunk_end2 = min(items, it2 + kChunk);
        if (it2 < items) tile_of(it2, ca2, st2);
      } else {
        it2 = it1 + 1;
        walk(ca1, st1, ca2, st2);
      }
    }
    if (tid == 0) {
      const uint32_t id = idesc_tf32(kTM, a.NT);
#pragma unroll
      for (int h = 0; h < TP / kTM; ++h) {   // the CTA's 128-point tiles, one accumulator each
        const uint32_t sa = smem_u32(sA) + (uint32_t)(h * kTM * a.Dp * 4);
        for (int ks = 0; ks < a.Dp / 8; ++ks) {   // one MMA per 8 tf32 of K (two 16-byte chunks)
          const uint64_t da = umma_desc(sa + ks * 256, 128, KC * 128);
          const uint64_t db = umma_desc(smem_u32(sB) + ks * 256, 128, KC * 128);
          const uint32_t acc = ks > 0;
          asm volatile(
              "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
              "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + (uint32_t)(h * a.tmem_tile)),
              "l"(da), "l"(db), "r"(id), "r"(acc));
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(&bar))
                   : "memory");
    }
    // the index of the tile after next (its rows are copied one tile later)
    const int64_t gi2 = it2 < items ? load_idx(ca2, st2) : -1;
    mark(2);
    asm volatile(
        "{\n.reg .pred P1;\nTCW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra TCW_%=;\n}\n" ::"r"(
            smem_u32(&bar)),
        "r"(phase)
        : "memory");
    phase ^= 1u;
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // sA is free: the next tile's rows land during this tile's epilogue
    if (pref && it1 < items) copy_rows();
    mark(3);
    // ---- epilogue: thread tid owns point tid (TMEM lane tid % 128 of tile tid / 128); per column the fp32 lower
    // bound L_j of rho_j^2 (bound above), tracking the smallest (index b, its S) and the
    // second smallest
    // ||y||^2 as computed (fp32 sequential on the prefetch path, fp64 otherwise) and its
    // enclosure [Y2l, Y2u] with gamma = (K + 2) 2^-24
    const double Y2c = sY2[tid];
    const double gamY = (a.Dp + 2) * 0x1p-24;
    const double Y2u = Y2c * (1.0 + gamY), Y2l = Y2c * (1.0 - gamY);
    const double yn = (double)__fsqrt_ru(__double2float_ru(Y2u));   // >= ||y||
    const double dmx = u * (yn + s_ca_norm + s_zmax) + 0x1p-51 * Cm + 0x1p-120;
    const double Ea = (2.0 * eps_s * yn + 2.0 * dmx) * (1.0 + 1e-6);
    const double Eb0 = (2.0 * (yn + dmx) * dmx + dmx * dmx + 0x1p-100) * (1.0 + 1e-6);
    const float Eaf = __double2float_ru(Ea);
    const float V = __double2float_rd(Y2l * (1.0 - kKappa) - Eb0);
    // two independent chains (even / odd columns) for instruction-level parallelism; NT is k
    // rounded up to 16 (padding columns: L = +inf): 32-column loads, a 16-column tail
    ColTrack tr;
    const float4* sWZ2 = reinterpret_cast<const float4*>(sWZ);   // column pairs
    const uint32_t trow = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((tid / kTM) * a.tmem_tile);
    int c0 = 0;
    for (; c0 + 32 <= a.NT; c0 += 32) tc_columns<32>(trow + (uint32_t)c0, c0, sWZ2, Eaf, V, tr);
    if (c0 < a.NT) tc_columns<16>(trow + (uint32_t)c0, c0, sWZ2, Eaf, V, tr);
    const float L2 = fminf(fminf(tr.L2e, tr.L2o), fmaxf(tr.L1e, tr.L1o));
    const bool odd = tr.L1o < tr.L1e;
    const float Sb = odd ? tr.Sbo : tr.Sbe;
    const int b = odd ? tr.bo : tr.be;
    mark(4);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    if (tid < cnt) {
      const int64_t gi = gi_cur;
      bool ok = b >= 0 && Y2u < 1e30 && !s_zbad;
      double low = (double)INFINITY;
      if (ok) {
        // upper bound of rho_b^2 in fp64: D*_b + E_b with ||z_b||^2 <= fl32(.)(1 + 2^-23)
        const double Z2b = (double)sZ2f[b] * (1.0 + 0x1p-23);
        const double Sd = (double)Sb;
        const double up = (Y2u + Z2b - 2.0 * Sd + Ea * (double)sWZ[b].y + Eb0 +
                           0x1p-40 * (Y2u + Z2b + 2.0 * fabs(Sd))) * (1.0 + 1e-12) + 0x1p-100;
        if (a.k > 1) low = (double)L2 * (1.0 - 1e-12);
        ok = low > up;
      }
      if (ok) {
        // proven unique argmin; its exact distance with the scan's arithmetic (R8): computed
        // during staging when b == a (prefetch path), else by tc_fix_kernel
        a.lab[gi] = b;
        a.lo[gi] = isinf(low) ? (double)INFINITY : sqrt(low);
        if (pref && b == ca) a.dmin[gi] = acc_a;
        else a.fix[atomicAdd(a.fix_len, 1)] = static_cast<int32_t>(gi);
      } else {
        a.amb[atomicAdd(a.amb_len, 1)] = static_cast<int32_t>(gi);
      }
    }
    mark(5);
    __syncthreads();   // sA / TMEM / s_chunk reused by the next tile
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    it = it1;
    ca = ca1;
    start = st1;
    gi_cur = gi1;
    it1 = it2;
    ca1 = ca2;
    st1 = st2;
    chunk_end1 = chunk_end2;
    gi1 = gi2;
  }
  if (a.prof && tid == 0) {
    for (int i = 0; i < 7; ++i) atomicAdd(a.prof + i, pt[i]);
    atomicAdd(a.prof + 7, 1ull);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(a.tmem_cols));
}

// exact (R8) distance of the decided points whose winner is not their current cluster
__global__ void __launch_bounds__(256) tc_fix_kernel(const float* __restrict__ F, const double* __restrict__ C, int d,
                                                     int v4, const int32_t* __restrict__ lab,
                                                     const int32_t* __restrict__ fix, const int* __restrict__ fix_len,
                                                     double* __restrict__ dmin) {
  const int m = *fix_len;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const int64_t gi = fix[i];
    const double* c = C + (size_t)lab[gi] * d;
    const float* x = F + gi * d;
    double acc = 0.0;
    if (v4) {
      for (int q0 = 0; q0 < d; q0 += 4) {
        const float4 xv = __ldg(reinterpret_cast<const float4*>(x + q0));
        const float xs[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const double diff = __dsub_rn((double)xs[e], c[q0 + e]);
          acc = __dadd_rn(acc, __dmul_rn(diff, diff));
        }
      }
    } else {
      for (int q = 0; q < d; ++q) {
        const double diff = __dsub_rn((double)__ldg(x + q), c[q]);
        acc = __dadd_rn(acc, __dmul_rn(diff, diff));
      }
    }
    dmin[gi] = acc;
  }
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

// offsets (exclusive scan of the counts) and the tiles' prefix ioff (tiles of <= tp points
// of one cluster), cursors and counters zeroed; one block, k <= 256
__global__ void __launch_bounds__(256) group_plan_kernel(const unsigned* __restrict__ cnt, int k,
                                                         int64_t* __restrict__ off, unsigned* __restrict__ cursor,
                                                         int* __restrict__ ioff, int* __restrict__ n_items,
                                                         int* __restrict__ ctr, int* __restrict__ fix_len,
                                                         int tp) {
  __shared__ long long s_c[256];
  __shared__ int s_i[256];
  const int tid = threadIdx.x;
  const long long cc = tid < k ? (long long)cnt[tid] : 0;
  const int ni = (int)((cc + tp - 1) / tp);
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
  if (tid < k) {
    off[tid] = s_c[tid] - cc;
    ioff[tid] = s_i[tid] - ni;
    cursor[tid] = 0u;
  }
  if (tid == 0) {
    off[k] = s_c[255];
    ioff[k] = s_i[255];
    *n_items = s_i[255];
    *ctr = 0;
    *fix_len = 0;
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
  const int NT = (k + 15) / 16 * 16, Dp = (d + 7) / 8 * 8;
  const size_t smem = tc_smem_bytes(NT, Dp);
  return k >= 2 && NT <= 256 && smem <= 200 * 1024;
}

int tc_screen(const float* F, int64_t n, int d, const double* C, const float* Cf, const double* cm, int k,
              const int32_t* old_lab, const int32_t* list, const int* list_len, int32_t* lab, double* dmin,
              double* lo, int32_t* amb, int* amb_len, TcWork& w, cudaStream_t s) {
  const int NT = (k + 15) / 16 * 16, Dp = (d + 7) / 8 * 8;
  SC_TRY(w.cnt.ensure(sizeof(unsigned) * 2 * (size_t)k, s));
  SC_TRY(w.off.ensure(sizeof(int64_t) * (size_t)(k + 1), s));
  SC_TRY(w.items.ensure(sizeof(int) * ((size_t)k + 4), s));   // ioff[k + 1], n_items, ctr, fix_len
  SC_TRY(w.fix.ensure(sizeof(int32_t) * (size_t)std::max<int64_t>(1, n), s));
  const int panel_floats = NT * Dp + 3 * NT;
  SC_TRY(w.panels.ensure(sizeof(float) * (size_t)k * panel_floats, s));
  SC_TRY(w.pscal.ensure(sizeof(double) * 16 * (size_t)k, s));
  SC_TRY(w.gperm.ensure(sizeof(int32_t) * (size_t)std::max<int64_t>(1, n), s));
  unsigned* cnt = w.cnt.as<unsigned>();
  unsigned* cursor = cnt + k;
  int* n_items = w.items.as<int>() + (size_t)k + 1;
  int* ctr = n_items + 1;
  int* fix_len = n_items + 2;
  int sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // kernel attributes once per process and instantiation (thread-safe static initialisation:
  // restarts call this from several worker threads): the largest dynamic shared memory any
  // supported (k, d) needs (tc_screen_supported caps it at 200 KB), the full shared-memory
  // carve-out, and the registers per thread for the occupancy below
  auto attrs = [](auto kern) {
    cudaFuncAttributes f{};
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&f, kern);
    return std::make_pair(e, f);
  };
  static const std::pair<cudaError_t, cudaFuncAttributes> kattr = attrs(assign_tc_kernel<kPV, 3, kTM>);
  static const std::pair<cudaError_t, cudaFuncAttributes> kattr_w = attrs(assign_tc_kernel<kPVWide, 1, kTM>);
  static const std::pair<cudaError_t, cudaFuncAttributes> kattr_p = attrs(assign_tc_kernel<kPVWide, 1, 2 * kTM>);
  SC_CUDA_TRY(kattr.first);
  SC_CUDA_TRY(kattr_w.first);
  SC_CUDA_TRY(kattr_p.first);
  const int tmem_tile = NT <= 32 ? 32 : NT <= 64 ? 64 : NT <= 128 ? 128 : 256;
  const bool v4 = (d % 4 == 0) && ((uintptr_t)F % 16 == 0) && ((uintptr_t)Cf % 16 == 0);
  // resident CTAs per SM: shared memory (228 KB per SM, 1 KB reserved per CTA), registers and
  // TMEM (512 columns per SM), computed here: the occupancy API answered 1 for this kernel
  // where the hardware fits 3 (ncu "Block Limit Shared Mem" / "Block Limit Registers" = 3 / 4
  // at k = 100, d = 64)
  auto occupancy = [&](const cudaFuncAttributes& fa, int tp) {
    const int sm = (int)tc_smem_bytes(NT, Dp, tp);
    const int regs_cta = std::max(1, fa.numRegs) * tp;
    const int o = std::min((227 * 1024) / (sm + (int)fa.sharedSizeBytes + 1024), 65536 / regs_cta);
    return std::min(o, 512 / (tmem_tile * (tp / kTM)));
  };
  const int occ = std::max(1, occupancy(kattr.second, kTM));
  // rows of 17-32 16-byte chunks (64 < d <= 128) where shared memory or TMEM already allow one
  // CTA per SM only (configs[4]: k = 200, d = 96): the wide instantiation keeps the next tile's
  // rows in registers too, and, when two tiles' rows fit beside the panel, takes two tiles of
  // the cluster per CTA (8 warps per SM).  Env (tooling): SC_KMEANS_TC_WIDE=0 the narrow
  // kernel's staging loads, SC_KMEANS_TC_PAIR=0 one tile per CTA.
  auto env_on = [](const char* name) {
    const char* e = std::getenv(name);
    return !(e && std::atoi(e) == 0);
  };
  const int nval = d / 4;
  const bool wide = env_on("SC_KMEANS_TC_WIDE") && v4 && nval > kPV && nval <= kPVWide && occ == 1 &&
                    occupancy(kattr_w.second, kTM) == 1;
  const bool pair = wide && env_on("SC_KMEANS_TC_PAIR") && tc_smem_bytes(NT, Dp, 2 * kTM) <= 200 * 1024 &&
                    occupancy(kattr_p.second, 2 * kTM) == 1;
  const int TP = pair ? 2 * kTM : kTM;
  const int smem = (int)tc_smem_bytes(NT, Dp, TP);
  if (std::getenv("SC_KMEANS_TRACE"))
    std::fprintf(stderr, "[sc_kmeans] tensor screen: %d CTAs per SM, smem %d B%s%s\n", pair ? 1 : occ, smem,
                 wide ? ", wide prefetch" : "", pair ? ", two tiles per CTA" : "");
  const int max_items = (int)((n + TP - 1) / TP) + k;
  SC_CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(unsigned) * k, s));
  const int pgrid = (int)std::max<int64_t>(1, (n + kGChunk - 1) / kGChunk);   // (list: <= n entries)
  group_hist_kernel<<<pgrid, 256, sizeof(unsigned) * k, s>>>(old_lab, list, list_len, n, k, cnt);
  group_plan_kernel<<<1, 256, 0, s>>>(cnt, k, w.off.as<int64_t>(), cursor, w.items.as<int>(), n_items, ctr, fix_len, TP);
  tc_panel_kernel<<<dim3(k, (NT + 31) / 32), 256, 0, s>>>(C, k, d, Dp, NT, w.panels.as<float>(), w.pscal.as<double>(),
                                                    panel_floats);
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
  a.ioff = w.items.as<int>();
  a.n_items = n_items;
  a.goff = w.off.as<int64_t>();
  a.gperm = w.gperm.as<int32_t>();
  a.k = k;
  a.d = d;
  a.Dp = Dp;
  a.NT = NT;
  a.tmem_tile = tmem_tile;
  a.tmem_cols = tmem_tile * (TP / kTM);
  a.v4 = v4;
  a.panels = w.panels.as<float>();
  a.pscal = w.pscal.as<double>();
  a.panel_floats = panel_floats;
  a.ctr = ctr;
  // tooling (env SC_TC_PROFILE): per-phase cycle sums in managed memory, allocated once
  static const bool want_prof = std::getenv("SC_TC_PROFILE") != nullptr;
  static unsigned long long* const prof = [] {
    unsigned long long* q = nullptr;
    if (want_prof && cudaMallocManaged(&q, 8 * sizeof(unsigned long long)) != cudaSuccess) q = nullptr;
    if (q) std::memset(q, 0, 8 * sizeof(unsigned long long));
    return q;
  }();
  a.prof = prof;
  a.fix = w.fix.as<int32_t>();
  a.fix_len = fix_len;
  a.lab = lab;
  a.dmin = dmin;
  a.lo = lo;
  a.amb = amb;
  a.amb_len = amb_len;
  const int grid = (int)std::min<int64_t>(max_items, (int64_t)sms * (pair || wide ? 1 : occ));
  if (pair) assign_tc_kernel<kPVWide, 1, 2 * kTM><<<grid, 2 * kTM, smem, s>>>(a);
  else if (wide) assign_tc_kernel<kPVWide, 1, kTM><<<grid, kTM, smem, s>>>(a);
  else assign_tc_kernel<kPV, 3, kTM><<<grid, kTM, smem, s>>>(a);
  SC_CUDA_TRY(cudaGetLastError());
  tc_fix_kernel<<<sms * 2, 256, 0, s>>>(F, C, d, a.v4, lab, a.fix, fix_len, dmin);
  SC_CUDA_TRY(cudaGetLastError());
  if (prof) {   // tooling: per-phase cycles of thread 0, summed over CTAs and launches
    static std::atomic<int> calls{0};
    if (++calls % 200 == 0) {
      SC_CUDA_TRY(cudaStreamSynchronize(s));
      const double c = (double)std::max(1ull, prof[7]);
      std::fprintf(stderr, "[sc_kmeans] tensor screen cycles per CTA: next/panel %.0f stage %.0f mma+prefetch %.0f "
                   "wait %.0f columns %.0f decide %.0f end %.0f\n", prof[0] / c, prof[1] / c, prof[2] / c, prof[3] / c,
                   prof[4] / c, prof[5] / c, prof[6] / c);
    }
  }
  return SC_OK;
}

}  // namespace sc
