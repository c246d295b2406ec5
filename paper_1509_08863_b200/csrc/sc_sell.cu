// Fused Chebyshev recurrence step over a sliced, padded copy of the CSR (SELL layout).
//
// PAPER.md §2.4 Eq. (3) (lines 135-147) and §4.1 step 5 Eq. (10) (line 321): the filter is
// p sparse products with L = S - W, run as the Chebyshev three-term recurrence
// (R1).  One launch = one step over one column chunk:
//     T_{s+1}[i] = a (s_i T_s[i] - sum_k W_ik T_s[k]) + b_cur T_s[i] + b_prev T_{s-1}[i]
//     Y[i]      (=|+=) cy_prev T_{s-1}[i] + cy_cur T_s[i] + cy_next T_{s+1}[i]
// (same arithmetic as cheb_step_kernel in sc_filter.cu, which stays for the moments and
// row-partitioned paths).
//
// Why a second layout.  cheb_step_kernel walks the plain CSR: every gathered 16-byte
// vector costs ~19 SASS instructions per lane (bounds tests per window slot, zero fills
// for lanes whose row ended, one index load per edge, four scalar adds), and on configs[3]
// the launch is issue-bound (ncu: issue active 74 %, 190 M warp instructions per launch).
// Here each tile's rows are cut into slices of RPW rows (the rows one warp processes
// together, already degree-sorted by tile_order), every row of a slice is padded to the
// slice's longest row rounded up to 4 with a sentinel column index that points at an
// all-zero row appended to the gathered block (row n_cols), and the indices are stored
// 4-edge-chunk-interleaved so one 16-byte shared-memory load gives a lane the next four
// column indices of its row without bank conflicts:
//     slice entry (row r of the slice, edge e) at  off + (e / 4) * 4 * RPW + 4 r + e % 4.
// The gather loop then has no per-edge predicate, no zero fill and a warp-uniform trip
// count; each gathered vector is one IMAD.WIDE + one LDG.E.128 + two packed FADD2
// (add.rn.f32x2), i.e. ~5 instructions per edge per lane.  Adding the padding's zero
// rows changes nothing (x + 0 = x), so the per-element sums are the CSR-order sums of
// cheb_step_kernel exactly.
//
// Build (once per graph and tile shape, cached on the handle): sell_len_kernel (padded
// slice lengths), a host prefix over tiles, sell_fill_kernel (slice metadata + entries).
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "sc_internal.cuh"
#include "sc_ptx.cuh"

namespace sc {
namespace {

#ifndef SC_SELL_NC
#define SC_SELL_NC 16       // consumer warps per CTA (= slices per tile)
#endif
#ifndef SC_SELL_MIN_CTAS
#define SC_SELL_MIN_CTAS 2  // resident CTAs per SM the register budget is sized for
#endif
#ifndef SC_SELL_NB
#define SC_SELL_NB 1        // 4-edge batches in flight per lane (configs[3], 32-column chunks:
#endif                      // 1 -> 97.1 ms per pass, 2 -> 107.1 ms; profiles/r02_sell.md)
#ifndef SC_SELL_NB_W
#define SC_SELL_NB_W 1      // weighted graphs
#endif
#ifndef SC_SELL_NB_F64
#define SC_SELL_NB_F64 1    // fp64 (configs[3], 16-double chunks: 1 -> 198.5 ms, 2 -> 219.6 ms)
#endif
#ifndef SC_SELL_STAGES
#define SC_SELL_STAGES 3
#endif
#ifndef SC_SELL_GATHER_L1
#define SC_SELL_GATHER_L1 0   // gathers: 0 ld.global.nc, 1 ld.global.nc.L1::no_allocate, 2 ld.global.cg
#endif
#ifndef SC_SELL_SMEM_TARGET_KB
#define SC_SELL_SMEM_TARGET_KB 80   // a plan's shared memory per CTA should stay at or below this:
#endif                              // the rest of the SM's 228 KB is L1, which holds the gathers in
                                    // flight (configs[3]: 16-column chunks 215 ms with 105 KB per
                                    // CTA, 123 ms with 54 KB; profiles/r02_sell.md)
#ifndef SC_SELL_SMEM_KB
#define SC_SELL_SMEM_KB 113   // most shared memory per CTA (2 CTAs per SM); a plan takes only
#endif                        // what its largest tile needs, the rest of the SM's 228 KB is L1
#if SC_SELL_GATHER_L1 == 1
#define SC_GLD "ld.global.nc.L1::no_allocate"
#elif SC_SELL_GATHER_L1 == 2
#define SC_GLD "ld.global.cg"
#else
#define SC_GLD "ld.global.nc"
#endif
constexpr int kNC = SC_SELL_NC;
constexpr int kThreads = (kNC + 1) * 32;
constexpr int kStages = SC_SELL_STAGES;   // most stages a plan uses
static_assert(kStages <= 4, "header holds at most 4 stages");

struct SellTileMeta {
  int64_t r0, r1;     // rows [r0, r1); r0 < 0: no more tiles
  int64_t e0;         // first SELL entry of the tile
  int32_t overflow;   // 1: the tile's entries did not fit the stage, read them from global
  int32_t tile;
};

__host__ __device__ constexpr int sell_tile_rows(int vpr) { return kNC * (32 / vpr); }

struct SellLayout {
  int cap;   // SELL entries per stage
  size_t meta_off, ord_off, idx_off, val_off, stage_bytes, dense_off, total;
  // stages: CSR ring depth (2..kStages); dense: own / T_{s-1} / Y rows staged with cp.async
  // during the gathers (else plain loads after the gather loop: less shared memory)
  __host__ __device__ SellLayout(int tr, int cap_, bool unit, int stages, bool dense) {
    cap = cap_;
    meta_off = 0;
    ord_off = (size_t)kNC * 16;
    idx_off = ord_off + (((size_t)tr * 4 + 15) & ~(size_t)15);
    val_off = idx_off + (size_t)cap * 4;
    stage_bytes = val_off + (unit ? 0 : (size_t)cap * 4);
    stage_bytes = (stage_bytes + 127) & ~(size_t)127;
    dense_off = 256 + (size_t)stages * stage_bytes;
    total = dense_off + (dense ? (size_t)kNC * 3 * 32 * 16 : 0);
  }
};

struct SellDev {
  const int64_t* tile_ptr;   // [ntiles + 1] first entry of each tile (multiple of 4)
  const int4* meta;          // [ntiles * kNC] per slice: {offset in the tile, padded length,
                             //   hub mask (bit r: slice row r is a hub), first hub id}
  const int32_t* hub_chunk_ptr;   // [n_hubs + 1] chunks of each hub row (split-row path)
  const void* hubpart;            // [n_chunks][width] partial sums of the hub chunks (type T)
  const int32_t* idx;        // column indices (sentinel n_cols = the zero row)
  const float* val;          // weights (0 on padding), nullptr for unit weights
  const int32_t* order;      // [ntiles * tr] row (relative to row_begin) at each tile position:
                             // degree-sorted within windows of sigma rows (SELL-C-sigma)
};

// 16-byte gathers as two packed fp32 pairs (for add.rn.f32x2)
__device__ __forceinline__ void ldg_pair2(const void* p, uint64_t& a, uint64_t& b) {
  asm volatile(SC_GLD ".v2.b64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "l"(p));
}
__device__ __forceinline__ void add_f32x2(uint64_t& acc, uint64_t v) {
  asm("add.rn.f32x2 %0, %0, %1;" : "+l"(acc) : "l"(v));
}
__device__ __forceinline__ void ldg_d2(const void* p, double& a, double& b) {
  asm volatile(SC_GLD ".v2.f64 {%0,%1}, [%2];" : "=d"(a), "=d"(b) : "l"(p));
}
__device__ __forceinline__ void ldg_f4(const void* p, float& a, float& b, float& c, float& d) {
  asm volatile(SC_GLD ".v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(a), "=f"(b), "=f"(c), "=f"(d) : "l"(p));
}

// Sum of the gathered rows of one lane's row: acc[w] += T_s[k][c + w] (x weight), over the
// padded slice row, NB 4-edge batches in flight.  `ci` / `cw`: this lane's first 4-index
// chunk (chunk b at ci + b * 4 * RPW).  Warp-uniform trip count nb = padded length / 4.
// Loads are unconditional (a conditional load would keep the slot's previous value live
// across it); a lane without a row passes ldb = 0, so its loads all hit one L1 line.
template <typename T, int RPW, int NB, bool UNIT> struct Gather;

template <int RPW, int NB> struct Gather<float, RPW, NB, true> {
  static __device__ __forceinline__ void run(const int32_t* __restrict__ ci, const float* __restrict__,
                                             int nb, const char* gbase, uint32_t ldb, float (&acc)[4]) {
    constexpr int CS = 4 * RPW;
    uint64_t a0 = 0, a1 = 0;
    uint64_t g[NB][4][2];
    auto issue = [&](int slot, int b) {
      const int4 k = *reinterpret_cast<const int4*>(ci + b * CS);
      {
        ldg_pair2(gbase + (uint64_t)(uint32_t)k.x * ldb, g[slot][0][0], g[slot][0][1]);
        ldg_pair2(gbase + (uint64_t)(uint32_t)k.y * ldb, g[slot][1][0], g[slot][1][1]);
        ldg_pair2(gbase + (uint64_t)(uint32_t)k.z * ldb, g[slot][2][0], g[slot][2][1]);
        ldg_pair2(gbase + (uint64_t)(uint32_t)k.w * ldb, g[slot][3][0], g[slot][3][1]);
      }
    };
#pragma unroll
    for (int s = 0; s < NB; ++s)
      if (s < nb) issue(s, s);
    for (int b0 = 0; b0 < nb; b0 += NB) {
#pragma unroll
      for (int s = 0; s < NB; ++s) {
        if (b0 + s < nb) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            add_f32x2(a0, g[s][e][0]);
            add_f32x2(a1, g[s][e][1]);
          }
          if (b0 + s + NB < nb) issue(s, b0 + s + NB);
        }
      }
    }
    acc[0] = __uint_as_float(static_cast<uint32_t>(a0));
    acc[1] = __uint_as_float(static_cast<uint32_t>(a0 >> 32));
    acc[2] = __uint_as_float(static_cast<uint32_t>(a1));
    acc[3] = __uint_as_float(static_cast<uint32_t>(a1 >> 32));
  }
};

template <int RPW, int NB> struct Gather<float, RPW, NB, false> {
  static __device__ __forceinline__ void run(const int32_t* __restrict__ ci, const float* __restrict__ cw,
                                             int nb, const char* gbase, uint32_t ldb, float (&acc)[4]) {
    constexpr int CS = 4 * RPW;
    float g[NB][4][4];
    acc[0] = acc[1] = acc[2] = acc[3] = 0.f;
    auto issue = [&](int slot, int b) {
      const int4 k = *reinterpret_cast<const int4*>(ci + b * CS);
      {
        ldg_f4(gbase + (uint64_t)(uint32_t)k.x * ldb, g[slot][0][0], g[slot][0][1], g[slot][0][2], g[slot][0][3]);
        ldg_f4(gbase + (uint64_t)(uint32_t)k.y * ldb, g[slot][1][0], g[slot][1][1], g[slot][1][2], g[slot][1][3]);
        ldg_f4(gbase + (uint64_t)(uint32_t)k.z * ldb, g[slot][2][0], g[slot][2][1], g[slot][2][2], g[slot][2][3]);
        ldg_f4(gbase + (uint64_t)(uint32_t)k.w * ldb, g[slot][3][0], g[slot][3][1], g[slot][3][2], g[slot][3][3]);
      }
    };
#pragma unroll
    for (int s = 0; s < NB; ++s)
      if (s < nb) issue(s, s);
    for (int b0 = 0; b0 < nb; b0 += NB) {
#pragma unroll
      for (int s = 0; s < NB; ++s) {
        if (b0 + s < nb) {
          // weights read from the staged segment when consumed (no registers held)
          const float4 wv = *reinterpret_cast<const float4*>(cw + (b0 + s) * CS);
          const float w4[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
          for (int e = 0; e < 4; ++e)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[q] = fmaf(w4[e], g[s][e][q], acc[q]);
          if (b0 + s + NB < nb) issue(s, b0 + s + NB);
        }
      }
    }
  }
};

template <int RPW, int NB, bool UNIT> struct Gather<double, RPW, NB, UNIT> {
  static __device__ __forceinline__ void run(const int32_t* __restrict__ ci, const float* __restrict__ cw,
                                             int nb, const char* gbase, uint32_t ldb, double (&acc)[2]) {
    constexpr int CS = 4 * RPW;
    double g[NB][4][2];
    acc[0] = acc[1] = 0.0;
    auto issue = [&](int slot, int b) {
      const int4 k = *reinterpret_cast<const int4*>(ci + b * CS);
      {
        ldg_d2(gbase + (uint64_t)(uint32_t)k.x * ldb, g[slot][0][0], g[slot][0][1]);
        ldg_d2(gbase + (uint64_t)(uint32_t)k.y * ldb, g[slot][1][0], g[slot][1][1]);
        ldg_d2(gbase + (uint64_t)(uint32_t)k.z * ldb, g[slot][2][0], g[slot][2][1]);
        ldg_d2(gbase + (uint64_t)(uint32_t)k.w * ldb, g[slot][3][0], g[slot][3][1]);
      }
    };
#pragma unroll
    for (int s = 0; s < NB; ++s)
      if (s < nb) issue(s, s);
    for (int b0 = 0; b0 < nb; b0 += NB) {
#pragma unroll
      for (int s = 0; s < NB; ++s) {
        if (b0 + s < nb) {
          if (UNIT) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              acc[0] += g[s][e][0];
              acc[1] += g[s][e][1];
            }
          } else {
            const float4 wv = *reinterpret_cast<const float4*>(cw + (b0 + s) * CS);
            const double w4[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              acc[0] = fma(w4[e], g[s][e][0], acc[0]);
              acc[1] = fma(w4[e], g[s][e][1], acc[1]);
            }
          }
          if (b0 + s + NB < nb) issue(s, b0 + s + NB);
        }
      }
    }
  }
};

// Fixed-point image of a moment partial for the order-independent sums: v x 2^80 truncated
// toward zero to a signed 128-bit integer (hi x 2^64 + lo), returned as limb `l` (32 bits) of its
// two's complement.  |v| < 2^47 (moment partials are bounded by ||X||_F^2).  The magnitude is
// split exactly (r = a - hi 2^64 is exact: a itself when hi = 0, Sterbenz when hi >= 1), then
// negated in 128-bit arithmetic.
__device__ __forceinline__ unsigned long long mom_limb(double v, int l) {
  const double a = fabs(v) * 0x1.0p80;
  const double hi = floor(a * 0x1.0p-64);
  const double r = a - hi * 0x1.0p64;          // exact, in [0, 2^64)
  unsigned long long lo = __double2ull_rz(r);
  unsigned long long h = __double2ull_rz(hi);
  if (v < 0.0) {                               // two's complement of (h, lo)
    lo = ~lo + 1ull;
    h = ~h + (lo == 0ull ? 1ull : 0ull);
  }
  const unsigned long long w = (l < 2) ? lo : h;
  return (l & 1) ? (w >> 32) : (w & 0xffffffffull);
}

template <typename T, int VPR, int NB, bool UNIT, bool P2P, bool MOM>
__global__ void __launch_bounds__(kThreads, SC_SELL_MIN_CTAS)
cheb_sell_kernel(SellDev sd, const T* __restrict__ strength, StepParams p, int cap, int cfg) {
  constexpr int W = Vec<T>::W;
  constexpr int SW = VPR;          // lanes per row (one 16-byte vector each)
  constexpr int RPW = 32 / SW;     // rows per warp = rows per slice
  constexpr int TR = sell_tile_rows(VPR);
  const int S = cfg & 15;                  // CSR ring stages
  const bool dense_stage = (cfg >> 4) & 1;  // cp.async staging of the dense rows

  extern __shared__ __align__(128) unsigned char smem[];
  const SellLayout lay(TR, cap, UNIT, S, dense_stage);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + 4;
  SellTileMeta* meta = reinterpret_cast<SellTileMeta*>(smem + 64);
  unsigned char* stages = smem + 256;
  unsigned char* dense = smem + lay.dense_off;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nrows = p.row_end - p.row_begin;
  const int64_t ntiles = (nrows + TR - 1) / TR;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kNC);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  if (warp == kNC) {
    // ------------------------------------------------------------- producer
    // tiles from the launch's counter (dynamic) or round-robin; a stage with r0 = -1 stops
    // the consumers.  The producer that makes the counter's last increment of the launch
    // (value ntiles + gridDim.x - 1) resets it to 0, so a counter slot is reusable by a
    // later launch (or a CUDA graph replay) without a host-side memset.
    int i = 0;
    if (lane == 0) {
      for (;; ++i) {
        const int s = i % S;
        int64_t t;
        if (p.tile_ctr) {
          const unsigned v = atomicAdd(p.tile_ctr, 1u);
          if ((int64_t)v == ntiles + gridDim.x - 1) atomicExch(p.tile_ctr, 0u);
          t = v;
        } else {
          t = blockIdx.x + (int64_t)i * gridDim.x;
        }
        if (i >= S) mbar_wait(&empty[s], ((i / S) - 1) & 1);
        SellTileMeta& m = meta[s];
        if (t >= ntiles) {
          m.r0 = -1;
          mbar_arrive(&full[s]);
          break;
        }
        const int64_t r0 = p.row_begin + t * TR;
        const int64_t r1 = min(r0 + TR, p.row_end);
        const int64_t e0 = __ldg(sd.tile_ptr + t), e1 = __ldg(sd.tile_ptr + t + 1);
        const int64_t ncol = e1 - e0;
        const int overflow = ncol > lay.cap;
        m.r0 = r0; m.r1 = r1; m.e0 = e0; m.overflow = overflow; m.tile = (int32_t)t;
        unsigned char* st = stages + (size_t)s * lay.stage_bytes;
        uint32_t tx = (uint32_t)(kNC * 16) + (uint32_t)(TR * 4);
        const bool cp_col = !overflow && ncol > 0;
        if (cp_col) tx += (uint32_t)(ncol * 4 * (UNIT ? 1 : 2));
        mbar_arrive_expect_tx(&full[s], tx);
        const uint64_t pol_stream = policy_evict_first();
        bulk_g2s(st + lay.meta_off, sd.meta + t * kNC, (uint32_t)(kNC * 16), &full[s], pol_stream);
        bulk_g2s(st + lay.ord_off, sd.order + t * TR, (uint32_t)(TR * 4), &full[s], pol_stream);
        if (cp_col) {
          bulk_g2s(st + lay.idx_off, sd.idx + e0, (uint32_t)(ncol * 4), &full[s], pol_stream);
          if (!UNIT) bulk_g2s(st + lay.val_off, sd.val + e0, (uint32_t)(ncol * 4), &full[s], pol_stream);
        }
      }
      // drain: wait until the consumers released every real tile's stage still in use
      for (int j = max(0, i - S); j < i; ++j) mbar_wait(&empty[j % S], (j / S) & 1);
    }
    __syncwarp();
    return;
  }

  // --------------------------------------------------------------- consumers
  asm volatile("griddepcontrol.wait;" ::: "memory");   // the previous step has completed
  const int sub = lane / SW;
  const int sl = lane % SW;
  const int c = sl * W;
  const T* tprev = static_cast<const T*>(p.tprev);   // may alias tnext (same row, read before write)
  const T* __restrict__ tcur = static_cast<const T*>(p.tcur);
  T* tnext = static_cast<T*>(p.tnext);
  T* y = static_cast<T*>(p.y);
  const char* gbase = reinterpret_cast<const char*>(tcur + c);
  const uint32_t ldb = static_cast<uint32_t>(p.ld_cur * sizeof(T));
  T* d_own = reinterpret_cast<T*>(dense + ((size_t)(warp * 3 + 0) * 32 + lane) * 16);
  T* d_prv = reinterpret_cast<T*>(dense + ((size_t)(warp * 3 + 1) * 32 + lane) * 16);
  T* d_y = reinterpret_cast<T*>(dense + ((size_t)(warp * 3 + 2) * 32 + lane) * 16);
  // MOM: lane l < 12 accumulates limb l % 4 of moment sum l / 4 over the warp's tiles (exact
  // integer adds: the result does not depend on which tiles the warp got)
  unsigned long long mom_acc = 0;

  for (int i = 0;; ++i) {
    const int s = i % S;
    mbar_wait(&full[s], (i / S) & 1);
    const SellTileMeta m = meta[s];
    if (m.r0 < 0) break;
    const int64_t t = m.tile;
    const unsigned char* st = stages + (size_t)s * lay.stage_bytes;
    // this warp's slice: one block of RPW consecutive degree ranks, the block index rotating
    // with the tile so every warp sees every degree class
    const int j = (warp + static_cast<int>(t % kNC)) % kNC;
    const int4 mj = reinterpret_cast<const int4*>(st + lay.meta_off)[j];
    const int32_t* ord = reinterpret_cast<const int32_t*>(st + lay.ord_off);
    const int rank = j * RPW + sub;
    const bool valid = sub < RPW && rank < static_cast<int>(m.r1 - m.r0);
    const int32_t row = static_cast<int32_t>(p.row_begin) + (valid ? ord[rank] : 0);   // rows < 2^31
    if (dense_stage && valid) {
      // own row, T_{s-1} and Y rows land in shared memory while the gathers run.  No L2
      // cache hint here: with one, ptxas 12.9 allocated the hint's 64-bit descriptor to an
      // odd uniform register (desc[UR1]) in the unit-weight instantiations, which faults with
      // cudaErrorIllegalInstruction (native_build.py now rejects such SASS)
      cp_async16_nohint(d_own, tcur + (int64_t)row * p.ld_cur + c);
      if (tprev) cp_async16_nohint(d_prv, tprev + (int64_t)row * p.ld_prev + c);
      if (p.y_mode == 2) cp_async16_nohint(d_y, y + (int64_t)row * p.ld_y + c);
    }
    const int lsub = sub < RPW ? sub : 0;
    double m_cc = 0.0, m_nc = 0.0, m_nn = 0.0;   // MOM: this lane's terms of the tile
    T acc[W];
    {
      // every tile fits a stage (launch_sell_step checks the plan's largest tile)
      const int32_t* ci = reinterpret_cast<const int32_t*>(st + lay.idx_off) + mj.x + 4 * lsub;
      const float* cw = reinterpret_cast<const float*>(st + lay.val_off) + mj.x + 4 * lsub;
      Gather<T, RPW, NB, UNIT>::run(ci, cw, mj.y >> 2, gbase, valid ? ldb : 0u, acc);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);

    if (p.split_mode == 1) {
      // first half of the columns: park the row sums, no epilogue (the second launch adds them)
      if (valid) Vec<T>::st(static_cast<T*>(p.split_buf) + (int64_t)row * p.width + c, acc);
      continue;
    }
    if (valid && ((mj.z >> sub) & 1)) {
      // a hub row (degree above the plan's threshold): its slice entries are empty and its
      // neighbour sum was split over warps by hub_chunk_kernel (launched just before, so
      // griddepcontrol.wait covered it); add the chunk partials in chunk order
      const int h = mj.w + __popc(static_cast<unsigned>(mj.z) & ((1u << sub) - 1u));
      const int c0 = sd.hub_chunk_ptr[h], c1 = sd.hub_chunk_ptr[h + 1];
      const T* hp = static_cast<const T*>(sd.hubpart) + c;
#pragma unroll
      for (int w = 0; w < W; ++w) acc[w] = T(0);
      for (int q = c0; q < c1; ++q) {
        T v[W];
        Vec<T>::ld(hp + (int64_t)q * p.width, v);
#pragma unroll
        for (int w = 0; w < W; ++w) acc[w] += v[w];
      }
    }
    if (valid && p.split_mode == 2) {
      // second half: + the first half's row sums (hub rows: 0 there, their sum came above)
      T pv[W];
      Vec<T>::ld(static_cast<const T*>(p.split_buf) + (int64_t)row * p.width + c, pv);
#pragma unroll
      for (int w = 0; w < W; ++w) acc[w] += pv[w];
    }
    if (valid) {
      T own[W], prv[W], yv[W];
      if (dense_stage) {
        asm volatile("cp.async.wait_all;" ::: "memory");
        Vec<T>::ld(d_own, own);
        if (tprev) Vec<T>::ld(d_prv, prv);
        if (p.y_mode == 2) Vec<T>::ld(d_y, yv);
      } else {
        const uint64_t pol = policy_evict_first();
        Vec<T>::ldg(tcur + (int64_t)row * p.ld_cur + c, own);
        if (tprev) Stream<T>::ld(tprev + (int64_t)row * p.ld_prev + c, prv, pol);
        if (p.y_mode == 2) Stream<T>::ld(y + (int64_t)row * p.ld_y + c, yv, pol);
      }
      if (!tprev) {
#pragma unroll
        for (int w = 0; w < W; ++w) prv[w] = T(0);
      }
      if (p.y_mode != 2) {
#pragma unroll
        for (int w = 0; w < W; ++w) yv[w] = T(0);
      }
      const T si = strength[row];
      const T a = static_cast<T>(p.a), bc = static_cast<T>(p.b_cur), bp = static_cast<T>(p.b_prev);
      T tn[W];
#pragma unroll
      for (int w = 0; w < W; ++w) {
        const T lt = si * own[w] - acc[w];               // (L T_s)[i]
        tn[w] = a * lt + bc * own[w] + bp * prv[w];      // T_{s+1}[i]
      }
      if (tnext) Vec<T>::st(tnext + (int64_t)row * p.ld_next + c, tn);   // gathered next step: normal L2 policy
      if (p.y_mode) {
        const T cyp = static_cast<T>(p.cy_prev), cyc = static_cast<T>(p.cy_cur), cyn = static_cast<T>(p.cy_next);
#pragma unroll
        for (int w = 0; w < W; ++w) yv[w] += cyp * prv[w] + cyc * own[w] + cyn * tn[w];
        Stream<T>::st(y + (int64_t)row * p.ld_y + c, yv, policy_evict_first());
      }
      if (P2P && tnext && row >= p.p2p->row0) {
        // fused halo exchange (multi-GPU): the peers that read this row get it straight into
        // their halo rows of the same buffer (NVLink stores from the epilogue)
        const P2PDev* x = p.p2p;
        const int64_t e1 = x->sd_ptr[row + 1];
        for (int64_t e = x->sd_ptr[row]; e < e1; ++e) {
          const int q = x->sd_peer[e];
          T* dst = static_cast<T*>(x->peer_buf[p.p2p_next][q]) + (x->peer_nl[q] + x->sd_slot[e]) * p.ld_next + c;
          Vec<T>::st(dst, tn);
        }
      }
      if (MOM) {
#pragma unroll
        for (int w = 0; w < W; ++w) {
          m_cc += (double)own[w] * (double)own[w];
          m_nc += (double)tn[w] * (double)own[w];
          m_nn += (double)tn[w] * (double)tn[w];
        }
      }
    }
    if (MOM) {
      // the warp's tile partial (fixed shuffle order), then its fixed-point limbs
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        m_cc += __shfl_xor_sync(0xffffffffu, m_cc, o);
        m_nc += __shfl_xor_sync(0xffffffffu, m_nc, o);
        m_nn += __shfl_xor_sync(0xffffffffu, m_nn, o);
      }
      const int comp = lane >> 2;
      const double v = comp == 0 ? m_cc : (comp == 1 ? m_nc : m_nn);
      if (lane < 12) mom_acc += mom_limb(v, lane & 3);
      m_cc = m_nc = m_nn = 0.0;
    }
  }

  if (MOM) {
    // CTA: the warps' limbs added in shared memory (integers: any order), then one global add
    // per limb
    __shared__ unsigned long long s_mom[12];
    if (threadIdx.x < 12) s_mom[threadIdx.x] = 0ull;
    asm volatile("bar.sync 3, %0;" ::"r"(kNC * 32) : "memory");
    if (lane < 12) atomicAdd(&s_mom[lane], mom_acc);
    asm volatile("bar.sync 3, %0;" ::"r"(kNC * 32) : "memory");
    if (threadIdx.x < 12) atomicAdd(p.mom_limbs + threadIdx.x, s_mom[threadIdx.x]);
  }
  if (P2P) {
    // publish completion to the peers (as cheb_step_kernel): every consumer thread fences its
    // remote stores, the last CTA to finish writes p2p_signal into each peer's flags (release)
    __threadfence_system();
    asm volatile("bar.sync 2, %0;" ::"r"(kNC * 32) : "memory");
    if (threadIdx.x == 0) {
      const P2PDev* x = p.p2p;
      if (atomicAdd(x->done_ctr, 1u) == gridDim.x - 1) {
        *x->done_ctr = 0u;
        __threadfence_system();
        for (int q = 0; q < x->world; ++q)
          if (q != x->rank)
            asm volatile("st.release.sys.global.b64 [%0], %1;" ::"l"(x->peer_flags[q] + x->rank), "l"(p.p2p_signal)
                         : "memory");
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Split rows (degree-adaptive traversal, north_star "chosen for the degree distribution";
// PAPER.md l.147 cost O(m(|E| + N))): a row whose degree exceeds the plan's threshold would
// pad its whole slice to its degree and be walked by one lane group (a straggler).  Its edges
// are cut into chunks of kHubChunk; one warp sums a chunk (its RPW lane groups take every
// RPW-th edge, then the groups are added in group order), the SELL kernel's epilogue adds the
// row's chunk partials in chunk order -- deterministic, and a hub costs as many warps as it
// has chunks.
// ---------------------------------------------------------------------------
#ifndef SC_HUB_CHUNK
#define SC_HUB_CHUNK 256   // Chung-Lu 127.4 (512) -> 126.2 ms (profiles/r02_hub3.txt)
#endif
constexpr int kHubChunk = SC_HUB_CHUNK;   // edges per split-row chunk (one warp each)
#ifndef SC_HUB_U
#define SC_HUB_U 4    // gathers in flight per lane in hub_chunk_kernel: Chung-Lu 143.0 / 133.9 / 129.4 /
#endif                // 129.6 ms per pass at 16 / 8 / 4 / 2 (profiles/r02_hub.txt, r02_hub2.txt); the
                      // launch caps at 16 blocks per SM (env SC_HUB_BPS; 8: 129.4, 16: 127.7 ms)
constexpr int kHubU = SC_HUB_U;

struct HubChunk {
  int64_t e0;     // first edge (CSR position)
  int32_t len;    // edges in the chunk
  int32_t pad;
};

template <typename T, int VPR, bool UNIT>
__global__ void __launch_bounds__(256)
hub_chunk_kernel(const HubChunk* __restrict__ chunks, int n_chunks, const int32_t* __restrict__ col,
                 const float* __restrict__ val, StepParams p, T* __restrict__ hubpart) {
  constexpr int W = Vec<T>::W;
  constexpr int SW = VPR;
  constexpr int RPW = 32 / SW;
  // the chunk's column indices (and weights) are staged in shared memory by the whole warp with
  // coalesced loads, so the gathers do not wait on a dependent index load
  __shared__ __align__(16) int32_t s_idx[8][kHubChunk];
  __shared__ __align__(16) float s_val[UNIT ? 1 : 8][UNIT ? 1 : kHubChunk];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int sub = lane / SW, sl = lane % SW, c = sl * W;
  const T* tcur = static_cast<const T*>(p.tcur);
  asm volatile("griddepcontrol.wait;" ::: "memory");
  for (int q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < n_chunks; q += (gridDim.x * blockDim.x) >> 5) {
    const HubChunk ch = chunks[q];
    __syncwarp();
    for (int e = lane; e < ch.len; e += 32) {
      s_idx[wib][e] = col[ch.e0 + e];
      if (!UNIT) s_val[wib][e] = val[ch.e0 + e];
    }
    __syncwarp();
    T acc[W];
#pragma unroll
    for (int w = 0; w < W; ++w) acc[w] = T(0);
    if (sub < RPW) {
      // kHubU gathers in flight per lane, added in edge order once the batch has landed
      for (int e0 = sub; e0 < ch.len; e0 += RPW * kHubU) {
        T v[kHubU][W];
        T wt[kHubU];
#pragma unroll
        for (int u = 0; u < kHubU; ++u) {
          const int e = e0 + u * RPW;
          if (e < ch.len) {
            const int64_t k = s_idx[wib][e];
            Vec<T>::ldg(tcur + k * p.ld_cur + c, v[u]);
            wt[u] = UNIT ? T(1) : static_cast<T>(s_val[UNIT ? 0 : wib][UNIT ? 0 : e]);
          } else {
#pragma unroll
            for (int w = 0; w < W; ++w) v[u][w] = T(0);
            wt[u] = T(0);
          }
        }
#pragma unroll
        for (int u = 0; u < kHubU; ++u)
#pragma unroll
          for (int w = 0; w < W; ++w) acc[w] = UNIT ? acc[w] + v[u][w] : fma(wt[u], v[u][w], acc[w]);
      }
    }
    // groups added in group order by the lanes of group 0
#pragma unroll
    for (int w = 0; w < W; ++w) {
      T tot = acc[w];
      for (int g = 1; g < RPW; ++g) {
        const T o = __shfl_sync(FULL, acc[w], sl + g * SW);
        tot += o;
      }
      acc[w] = tot;
    }
    if (sub == 0) Vec<T>::st(hubpart + (int64_t)q * p.width + c, acc);
  }
}

// ---------------------------------------------------------------------------
// SELL build
// ---------------------------------------------------------------------------
// Row order of the plan (SELL-C-sigma): rows sorted by degree (ascending, ties by index)
// within windows of sigma consecutive rows, hub rows (degree > hub_deg) last; tile t takes
// sorted positions [t tr, (t + 1) tr).  One block per window, bitonic sort in shared memory
// of keys degree << 32 | local index (unique).  Positions past the last row hold -1.
constexpr int kSigmaMax = 4096;

// edges of `row` with column in [c0, c1) (full = the whole row)
__device__ __forceinline__ int64_t deg_in(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                          int64_t row, int64_t c0, int64_t c1, bool full) {
  const int64_t b = rp[row], e = rp[row + 1];
  if (full) return e - b;
  int64_t d = 0;
  for (int64_t k = b; k < e; ++k) {
    const int64_t c = col[k];
    d += (c >= c0 && c < c1);
  }
  return d;
}
__global__ void __launch_bounds__(1024) sell_order_kernel(const int64_t* __restrict__ row_ptr,
                                                          const int32_t* __restrict__ col, int64_t c0, int64_t c1,
                                                          bool full, int64_t row_begin, int64_t row_end, int sigma,
                                                          int64_t hub_deg, int32_t* __restrict__ order) {
  __shared__ unsigned long long key[kSigmaMax];
  const int64_t w0 = row_begin + (int64_t)blockIdx.x * sigma;
  const int cnt = static_cast<int>(min((int64_t)sigma, row_end - w0));
  int P = 1;
  while (P < sigma) P <<= 1;
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    unsigned long long kk = ~0ull;
    if (i < cnt) {
      const int64_t d = row_ptr[w0 + i + 1] - row_ptr[w0 + i];   // hubs by their full degree
      const unsigned long long dk = d > hub_deg ? (unsigned long long)hub_deg + 1
                                                : (unsigned long long)deg_in(row_ptr, col, w0 + i, c0, c1, full);
      kk = (dk << 32) | (unsigned)i;
    }
    key[i] = kk;
  }
  __syncthreads();
  for (int k = 2; k <= P; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const int l = i ^ j;
        if (l > i) {
          const bool up = (i & k) == 0;
          const unsigned long long a = key[i], b = key[l];
          if ((a > b) == up) { key[i] = b; key[l] = a; }
        }
      }
      __syncthreads();
    }
  for (int i = threadIdx.x; i < sigma; i += blockDim.x)
    order[(int64_t)blockIdx.x * sigma + i] =
        i < cnt ? static_cast<int32_t>(w0 - row_begin + (int64_t)(unsigned)(key[i] & 0xffffffffull)) : -1;
}

// padded length of every slice (max degree of its rows rounded up to 4) and entries per tile
// (rows of degree > hub_deg are hubs: no slice entries, split-row path)
__global__ void sell_len_kernel(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col, int64_t c0,
                                int64_t c1, bool full, int64_t row_begin, int64_t row_end, int tr,
                                int rpw, const int32_t* __restrict__ order, int64_t hub_deg,
                                int32_t* __restrict__ slice_len, int64_t* __restrict__ tile_entries,
                                int32_t* __restrict__ tile_hubs) {
  const int64_t t = blockIdx.x;
  const int64_t r0 = row_begin + t * tr;
  const int cnt = static_cast<int>(min((int64_t)tr, row_end - r0));
  __shared__ int len[64], hubs[64];
  for (int j = threadIdx.x; j < kNC; j += blockDim.x) {
    int maxd = 0, nh = 0;
    for (int q = 0; q < rpw; ++q) {
      const int rank = j * rpw + q;
      if (rank < cnt) {
        const int64_t row = row_begin + order[t * tr + rank];
        const int64_t d = row_ptr[row + 1] - row_ptr[row];
        if (d > hub_deg) ++nh;
        else maxd = max(maxd, static_cast<int>(deg_in(row_ptr, col, row, c0, c1, full)));
      }
    }
    len[j] = (maxd + 3) & ~3;
    hubs[j] = nh;
    slice_len[t * kNC + j] = len[j];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t tot = 0;
    int nh = 0;
    for (int j = 0; j < kNC; ++j) {
      tot += (int64_t)len[j] * rpw;
      nh += hubs[j];
    }
    tile_entries[t] = tot;
    tile_hubs[t] = nh;
  }
}

__global__ void sell_fill_kernel(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                                 const float* __restrict__ val, int64_t c0, int64_t c1, bool full, int64_t row_begin,
                                 int64_t row_end, int tr, int rpw, const int32_t* __restrict__ order,
                                 const int32_t* __restrict__ slice_len, const int64_t* __restrict__ tile_ptr,
                                 int32_t sentinel, int64_t hub_deg, const int32_t* __restrict__ tile_hub_base,
                                 int4* __restrict__ meta, int32_t* __restrict__ idx, float* __restrict__ sval,
                                 int32_t* __restrict__ hub_rows) {
  const int64_t t = blockIdx.x;
  const int64_t r0 = row_begin + t * tr;
  const int cnt = static_cast<int>(min((int64_t)tr, row_end - r0));
  __shared__ int off[65];
  __shared__ int hub[1024];
  if (threadIdx.x == 0) {
    int o = 0;
    for (int j = 0; j < kNC; ++j) {
      off[j] = o;
      o += slice_len[t * kNC + j] * rpw;
    }
    off[kNC] = o;
  }
  for (int r = threadIdx.x; r < tr; r += blockDim.x) {
    hub[r] = 0;
    if (r < cnt) {
      const int64_t row = row_begin + order[t * tr + r];
      hub[r] = row_ptr[row + 1] - row_ptr[row] > hub_deg;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // hub ids in (tile, slice, slice row) order
    int h = tile_hub_base[t];
    for (int j = 0; j < kNC; ++j) {
      int mask = 0;
      const int base = h;
      for (int q = 0; q < rpw; ++q) {
        const int rank = j * rpw + q;
        if (rank < cnt && hub[rank]) {
          mask |= 1 << q;
          hub_rows[h++] = order[t * tr + rank];
        }
      }
      meta[t * kNC + j] = make_int4(off[j], slice_len[t * kNC + j], mask, base);
    }
  }
  // one thread per tile row: its edges in [c0, c1), in CSR order, at the chunk-interleaved
  // positions of its slice; the rest of the padded row gets the sentinel
  const int64_t base = tile_ptr[t];
  for (int rank = threadIdx.x; rank < kNC * rpw; rank += blockDim.x) {
    const int j = rank / rpw, q = rank % rpw;
    const int L = slice_len[t * kNC + j];
    int32_t* di = idx + base + off[j];
    float* dv = sval ? sval + base + off[j] : nullptr;
    int e = 0;
    if (rank < cnt && !hub[rank]) {
      const int64_t row = row_begin + order[t * tr + rank];
      for (int64_t k = row_ptr[row]; k < row_ptr[row + 1]; ++k) {
        const int64_t c = col[k];
        if (!full && (c < c0 || c >= c1)) continue;
        const int pos = (e / 4) * 4 * rpw + q * 4 + (e % 4);
        di[pos] = col[k];
        if (dv) dv[pos] = val[k];
        ++e;
      }
    }
    for (; e < L; ++e) {
      const int pos = (e / 4) * 4 * rpw + q * 4 + (e % 4);
      di[pos] = sentinel;
      if (dv) dv[pos] = 0.f;
    }
  }
}

struct SellPlan {
  int tr = 0, rpw = 0;
  int64_t ntiles = 0, entries = 0, max_tile = 0;
  DevBuf tile_ptr, meta, idx, val;
  DevBuf order;   // int32 [ntiles * tr]
  int sigma = 0;  // rows per degree-sorting window
  // split rows
  int64_t hub_deg = 0;
  int n_hubs = 0, n_chunks = 0;
  DevBuf hub_rows, hub_chunk_ptr, chunks, hubpart;
};

__global__ void max_degree_kernel(const int64_t* __restrict__ row_ptr, int64_t r0, int64_t r1,
                                  unsigned long long* __restrict__ out) {
  unsigned long long m = 0;
  for (int64_t i = r0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < r1; i += (int64_t)gridDim.x * blockDim.x)
    m = max(m, (unsigned long long)(row_ptr[i + 1] - row_ptr[i]));
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(FULL, m, o));
  if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

}  // namespace

int64_t max_row_degree(const sc_graph* g, int64_t r0, int64_t r1, cudaStream_t s) {
  DevBuf b;
  if (r1 <= r0 || b.ensure(sizeof(unsigned long long)) != SC_OK) return 0;
  unsigned long long h = 0;
  cudaMemsetAsync(b.ptr, 0, sizeof(h), s);
  max_degree_kernel<<<g->num_sms * 4, 256, 0, s>>>(g->row_ptr.as<int64_t>(), r0, r1, b.as<unsigned long long>());
  cudaMemcpyAsync(&h, b.ptr, sizeof(h), cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  return (int64_t)h;
}

namespace {

// split-row threshold: a row of degree > this is cut into chunks (env SC_SELL_HUB_DEG)
int64_t hub_threshold() {
  const char* v = std::getenv("SC_SELL_HUB_DEG");
  return v ? std::atoll(v) : 128;   // Chung-Lu (N = 10^6, exponent 2.1): 281 / 229 / 207 / 209 ms per
                                    // pass at 512 / 256 / 128 / 64 (profiles/r02_sell.md)
}

// hub rows' CSR ranges (device) -> host
__global__ void hub_range_kernel(const int64_t* __restrict__ row_ptr, int64_t row_begin, const int32_t* __restrict__ rows,
                                 int n, int64_t* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int64_t r = row_begin + rows[i];
    out[2 * i] = row_ptr[r];
    out[2 * i + 1] = row_ptr[r + 1];
  }
}

std::mutex g_sell_mu;
std::map<std::tuple<const sc_graph*, int, int64_t, int64_t, int64_t, int64_t>, std::unique_ptr<SellPlan>> g_sell_plans;

int env_int_s(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}

// Plan of the rows [row_begin, row_end) and the columns [c0, c1) (all columns: c0 = 0,
// c1 = n_cols; a column range keeps only those edges -- the split gather's halves)
int sell_plan(const sc_graph* g, int vpr, int64_t row_begin, int64_t row_end, cudaStream_t s, SellPlan** out,
              int64_t c0 = 0, int64_t c1 = -1) {
  const int tr = sell_tile_rows(vpr), rpw = 32 / vpr;
  if (c1 < 0) c1 = g->n_cols;
  const bool full = c0 <= 0 && c1 >= g->n_cols;
  std::lock_guard<std::mutex> lock(g_sell_mu);
  auto key = std::make_tuple(g, tr, row_begin, row_end, full ? 0 : c0, full ? g->n_cols : c1);
  auto it = g_sell_plans.find(key);
  if (it != g_sell_plans.end()) {
    *out = it->second.get();
    return SC_OK;
  }
  auto pl = std::make_unique<SellPlan>();
  pl->tr = tr;
  pl->rpw = rpw;
  pl->ntiles = (row_end - row_begin + tr - 1) / tr;
  const int64_t nt = pl->ntiles;
  pl->hub_deg = hub_threshold();
  // sorting window: one tile when the degrees are narrow (the tile's own sort pads little:
  // configs[3] 1.05), else up to kSigmaMax rows (power-law degrees: Chung-Lu padding
  // 1.38 -> 1.15 at 4096; env SC_SELL_SIGMA overrides)
  {
    const double avg = (double)g->nnz / std::max<int64_t>(1, g->n_rows);
    const int forced = env_int_s("SC_SELL_SIGMA", 0);
    int sig = tr;
    if (forced > 0) sig = std::max(tr, std::min(kSigmaMax, forced / tr * tr));
    else if ((double)max_row_degree(g, row_begin, row_end, s) > 8.0 * std::max(1.0, avg)) sig = kSigmaMax / tr * tr;
    pl->sigma = std::max(tr, sig);
  }
  SC_TRY(pl->order.ensure(sizeof(int32_t) * std::max<int64_t>(1, nt * tr)));
  if (nt > 0) {
    const int64_t nwin = (row_end - row_begin + pl->sigma - 1) / pl->sigma;
    // the last window's positions past nt * tr do not exist: sigma divides into whole tiles,
    // so allocate whole windows
    SC_TRY(pl->order.ensure(sizeof(int32_t) * (size_t)nwin * pl->sigma));
    sell_order_kernel<<<(unsigned)nwin, 1024, 0, s>>>(g->row_ptr.as<int64_t>(), g->col_idx.as<int32_t>(), c0, c1,
                                                      full, row_begin, row_end, pl->sigma, pl->hub_deg,
                                                      pl->order.as<int32_t>());
    SC_CUDA_TRY(cudaGetLastError());
  }
  DevBuf slen, tent, thub;
  SC_TRY(slen.ensure(sizeof(int32_t) * std::max<int64_t>(1, nt * kNC)));
  SC_TRY(tent.ensure(sizeof(int64_t) * std::max<int64_t>(1, nt)));
  SC_TRY(thub.ensure(sizeof(int32_t) * std::max<int64_t>(1, nt)));
  if (nt > 0) {
    sell_len_kernel<<<(unsigned)nt, 64, 0, s>>>(g->row_ptr.as<int64_t>(), g->col_idx.as<int32_t>(), c0, c1, full,
                                                row_begin, row_end, tr, rpw, pl->order.as<int32_t>(),
                                                pl->hub_deg, slen.as<int32_t>(), tent.as<int64_t>(),
                                                thub.as<int32_t>());
    SC_CUDA_TRY(cudaGetLastError());
  }
  std::vector<int64_t> h(nt), ptr(nt + 1, 0);
  std::vector<int32_t> th(nt), thb(nt + 1, 0);
  if (nt > 0) {
    SC_CUDA_TRY(cudaMemcpyAsync(h.data(), tent.ptr, sizeof(int64_t) * nt, cudaMemcpyDeviceToHost, s));
    SC_CUDA_TRY(cudaMemcpyAsync(th.data(), thub.ptr, sizeof(int32_t) * nt, cudaMemcpyDeviceToHost, s));
    SC_CUDA_TRY(cudaStreamSynchronize(s));
  }
  for (int64_t t = 0; t < nt; ++t) {
    ptr[t + 1] = ptr[t] + h[t];
    pl->max_tile = std::max(pl->max_tile, h[t]);
    thb[t + 1] = thb[t] + th[t];
  }
  pl->n_hubs = thb[nt];
  SC_TRY(pl->hub_rows.ensure(sizeof(int32_t) * std::max(1, pl->n_hubs)));
  DevBuf thbase;
  SC_TRY(thbase.ensure(sizeof(int32_t) * (nt + 1)));
  SC_CUDA_TRY(cudaMemcpyAsync(thbase.ptr, thb.data(), sizeof(int32_t) * (nt + 1), cudaMemcpyHostToDevice, s));
  pl->entries = ptr[nt];
  SC_TRY(pl->tile_ptr.ensure(sizeof(int64_t) * (nt + 1)));
  SC_CUDA_TRY(cudaMemcpyAsync(pl->tile_ptr.ptr, ptr.data(), sizeof(int64_t) * (nt + 1), cudaMemcpyHostToDevice, s));
  SC_TRY(pl->meta.ensure(sizeof(int4) * std::max<int64_t>(1, nt * kNC)));
  SC_TRY(pl->idx.ensure(sizeof(int32_t) * std::max<int64_t>(4, pl->entries)));
  if (!g->unit_weights) SC_TRY(pl->val.ensure(sizeof(float) * std::max<int64_t>(4, pl->entries)));
  if (nt > 0) {
    sell_fill_kernel<<<(unsigned)nt, 256, 0, s>>>(
        g->row_ptr.as<int64_t>(), g->col_idx.as<int32_t>(), g->unit_weights ? nullptr : g->values.as<float>(), c0,
        c1, full, row_begin, row_end, tr, rpw, pl->order.as<int32_t>(), slen.as<int32_t>(), pl->tile_ptr.as<int64_t>(),
        static_cast<int32_t>(g->n_cols), pl->hub_deg, thbase.as<int32_t>(), pl->meta.as<int4>(),
        pl->idx.as<int32_t>(), g->unit_weights ? nullptr : pl->val.as<float>(), pl->hub_rows.as<int32_t>());
    SC_CUDA_TRY(cudaGetLastError());
  }
  // split rows: chunks of kHubChunk edges per hub, in hub order
  std::vector<int32_t> cptr(pl->n_hubs + 1, 0);
  if (pl->n_hubs > 0) {
    DevBuf rng;
    SC_TRY(rng.ensure(sizeof(int64_t) * 2 * pl->n_hubs));
    hub_range_kernel<<<std::min(1024, (pl->n_hubs + 255) / 256), 256, 0, s>>>(
        g->row_ptr.as<int64_t>(), row_begin, pl->hub_rows.as<int32_t>(), pl->n_hubs, rng.as<int64_t>());
    SC_CUDA_TRY(cudaGetLastError());
    std::vector<int64_t> hr(2 * (size_t)pl->n_hubs);
    SC_CUDA_TRY(cudaMemcpyAsync(hr.data(), rng.ptr, sizeof(int64_t) * hr.size(), cudaMemcpyDeviceToHost, s));
    SC_CUDA_TRY(cudaStreamSynchronize(s));
    std::vector<HubChunk> ch;
    for (int hI = 0; hI < pl->n_hubs; ++hI) {
      for (int64_t e = hr[2 * hI]; e < hr[2 * hI + 1]; e += kHubChunk)
        ch.push_back(HubChunk{e, (int32_t)std::min<int64_t>(kHubChunk, hr[2 * hI + 1] - e), 0});
      cptr[hI + 1] = (int32_t)ch.size();
    }
    pl->n_chunks = (int)ch.size();
    SC_TRY(pl->chunks.ensure(sizeof(HubChunk) * std::max<size_t>(1, ch.size())));
    SC_CUDA_TRY(cudaMemcpyAsync(pl->chunks.ptr, ch.data(), sizeof(HubChunk) * ch.size(), cudaMemcpyHostToDevice, s));
  }
  SC_TRY(pl->hub_chunk_ptr.ensure(sizeof(int32_t) * (pl->n_hubs + 1)));
  SC_CUDA_TRY(cudaMemcpyAsync(pl->hub_chunk_ptr.ptr, cptr.data(), sizeof(int32_t) * (pl->n_hubs + 1),
                              cudaMemcpyHostToDevice, s));
  SC_CUDA_TRY(cudaStreamSynchronize(s));   // build temporaries are freed on return
  *out = pl.get();
  g_sell_plans[key] = std::move(pl);
  return SC_OK;
}

template <typename T>
using SellFn = void (*)(SellDev, const T*, StepParams, int, int);
template <typename T>
using HubFn = void (*)(const HubChunk*, int, const int32_t*, const float*, StepParams, T*);

template <typename T, int VPR>
HubFn<T> pick_hub_unit(bool unit) {
  return unit ? hub_chunk_kernel<T, VPR, true> : hub_chunk_kernel<T, VPR, false>;
}
template <typename T>
HubFn<T> pick_hub(int vpr, bool unit) {
  switch (vpr) {
    case 1: return pick_hub_unit<T, 1>(unit);
    case 2: return pick_hub_unit<T, 2>(unit);
    case 3: return pick_hub_unit<T, 3>(unit);
    case 4: return pick_hub_unit<T, 4>(unit);
    case 6: return pick_hub_unit<T, 6>(unit);
    case 8: return pick_hub_unit<T, 8>(unit);
    case 12: return pick_hub_unit<T, 12>(unit);
    case 16: return pick_hub_unit<T, 16>(unit);
    case 24: return pick_hub_unit<T, 24>(unit);
    default: return pick_hub_unit<T, 32>(unit);
  }
}

template <typename T, int VPR>
SellFn<T> pick_sell_unit(bool unit, bool p2p, bool mom) {
  // P2P: the fused-exchange epilogue of the row-partitioned fp32 path (a separate
  // instantiation: the single-GPU kernels keep their register allocation)
  // MOM: the eigencount moments (fp64 only)
  if constexpr (sizeof(T) == 4) {
    if (mom) return nullptr;
    if (p2p) return unit ? cheb_sell_kernel<T, VPR, SC_SELL_NB, true, true, false>
                         : cheb_sell_kernel<T, VPR, SC_SELL_NB_W, false, true, false>;
    if (unit) return cheb_sell_kernel<T, VPR, SC_SELL_NB, true, false, false>;
    return cheb_sell_kernel<T, VPR, SC_SELL_NB_W, false, false, false>;
  } else {
    if (p2p) return nullptr;
    if (mom) return unit ? cheb_sell_kernel<T, VPR, SC_SELL_NB_F64, true, false, true>
                         : cheb_sell_kernel<T, VPR, SC_SELL_NB_F64, false, false, true>;
    if (unit) return cheb_sell_kernel<T, VPR, SC_SELL_NB_F64, true, false, false>;
    return cheb_sell_kernel<T, VPR, SC_SELL_NB_F64, false, false, false>;
  }
}

template <typename T>
SellFn<T> pick_sell(int vpr, bool unit, bool p2p = false, bool mom = false) {
  switch (vpr) {
    case 1: return pick_sell_unit<T, 1>(unit, p2p, mom);
    case 2: return pick_sell_unit<T, 2>(unit, p2p, mom);
    case 3: return pick_sell_unit<T, 3>(unit, p2p, mom);
    case 4: return pick_sell_unit<T, 4>(unit, p2p, mom);
    case 6: return pick_sell_unit<T, 6>(unit, p2p, mom);
    case 8: return pick_sell_unit<T, 8>(unit, p2p, mom);
    case 12: return pick_sell_unit<T, 12>(unit, p2p, mom);
    case 16: return pick_sell_unit<T, 16>(unit, p2p, mom);
    case 24: return pick_sell_unit<T, 24>(unit, p2p, mom);
    case 32: return pick_sell_unit<T, 32>(unit, p2p, mom);
    default: return nullptr;
  }
}

// Launch configuration of a plan: stage capacity = its largest tile rounded up to 64
// entries; then the deepest CSR ring and the cp.async staging of the dense rows, in this order
// of preference, that keep the CTA at or below SC_SELL_SMEM_TARGET_KB (the rest of the SM's
// shared memory / L1 carve-out is L1, which holds the gathers in flight), else the smallest
// footprint; cap = 0 when even that exceeds SC_SELL_SMEM_KB.
struct SellCfg {
  int cap = 0, stages = 0;
  bool dense = false;
  size_t smem = 0;
  int packed() const { return stages | (dense ? 16 : 0); }
};
SellCfg sell_config(int tr, bool unit, int64_t max_tile) {
  SellCfg c;
  const int64_t cap = std::max<int64_t>(64, (max_tile + 63) & ~int64_t(63));
  if (cap > (int64_t)1 << 24) return c;
  const size_t target = (size_t)env_int_s("SC_SELL_SMEM_TARGET_KB", SC_SELL_SMEM_TARGET_KB) * 1024;
  const int forced_st = env_int_s("SC_SELL_FORCE_STAGES", 0), forced_dense = env_int_s("SC_SELL_FORCE_DENSE", -1);
  const struct { int st; bool dense; } order[] = {{3, true}, {2, true}, {3, false}, {2, false}};
  for (const auto& o : order) {
    if (o.st > kStages) continue;
    if (forced_st && o.st != forced_st) continue;
    if (forced_dense >= 0 && o.dense != (forced_dense != 0)) continue;
    const SellLayout lay(tr, (int)cap, unit, o.st, o.dense);
    if (lay.total > (size_t)SC_SELL_SMEM_KB * 1024) continue;
    c.cap = (int)cap;
    c.stages = o.st;
    c.dense = o.dense;
    c.smem = lay.total;
    if (lay.total <= target) break;   // first that meets the target; else keep the smallest
  }
  return c;
}

}  // namespace

bool sell_enabled() { return env_int_s("SC_SELL", 1) != 0; }   // read per call (tests switch it)

void sell_release(const sc_graph* g) {
  std::lock_guard<std::mutex> lock(g_sell_mu);
  for (auto it = g_sell_plans.begin(); it != g_sell_plans.end();) {
    if (std::get<0>(it->first) == g) it = g_sell_plans.erase(it);
    else ++it;
  }
}

// Can the SELL kernel run this (graph, chunk width, row range)?  Builds (and caches) the
// plan; false when a supported width has a tile whose padded entries exceed a stage (very
// high-degree rows: the CSR kernel handles those graphs).
template <typename T>
int sell_usable(const sc_graph* g, int width, int64_t row_begin, int64_t row_end, cudaStream_t s, bool* ok,
                int64_t split_col) {
  constexpr int W = Vec<T>::W;
  *ok = false;
  if (width % W || !pick_sell<T>(width / W, g->unit_weights) || row_end - row_begin >= INT_MAX) return SC_OK;
  const int vpr = width / W;
  SellPlan* pl = nullptr;
  if (split_col > 0) {
    SC_TRY(sell_plan(g, vpr, row_begin, row_end, s, &pl, 0, split_col));
    if (sell_config(sell_tile_rows(vpr), g->unit_weights, pl->max_tile).cap <= 0) return SC_OK;
    SC_TRY(sell_plan(g, vpr, row_begin, row_end, s, &pl, split_col, g->n_cols));
  } else {
    SC_TRY(sell_plan(g, vpr, row_begin, row_end, s, &pl));
  }
  *ok = sell_config(sell_tile_rows(vpr), g->unit_weights, pl->max_tile).cap > 0;
  return SC_OK;
}
template int sell_usable<float>(const sc_graph*, int, int64_t, int64_t, cudaStream_t, bool*, int64_t);
template int sell_usable<double>(const sc_graph*, int, int64_t, int64_t, cudaStream_t, bool*, int64_t);

// Split gather for this chunk?  The columns are gathered in two launches per step -- first
// [0, mid), row sums parked, then [mid, n_cols) and the epilogue -- each from half the table,
// meant for tables a little too big for L2 (configs[3], 32-column chunks: 128 MB in a 126 MB
// L2, ~68 % hit rate).  Measured slower everywhere (configs[3] 104.0 -> 136.8 ms per pass,
// fp64 201 -> 282 ms, weighted 104 -> 145 ms: each half pays the per-row work of all rows and
// the halves' degrees pad more), so it is off by default.  Returns the split column (0: none).
// env SC_SELL_SPLIT: 0 off (default), 1 auto (tables in (SC_SELL_SPLIT_MIN_MB,
// SC_SELL_SPLIT_MAX_MB]), 2 force.
int64_t sell_split_col(const sc_graph* g, int width, size_t elem) {
  const int mode = env_int_s("SC_SELL_SPLIT", 0);
  if (mode == 0) return 0;
  const double table = (double)g->n_cols * width * elem;
  const double lo = env_int_s("SC_SELL_SPLIT_MIN_MB", 96) * 1048576.0;
  const double hi = env_int_s("SC_SELL_SPLIT_MAX_MB", 160) * 1048576.0;
  if (mode == 2 || (table > lo && table <= hi)) return g->n_cols / 2;
  return 0;
}

// One fused step over the SELL layout.  Requirements: T_s (p.tcur) has a zero row at index
// g->n_cols (the sentinel of the padding); rows [row_begin, row_end) of one graph.
template <typename T>
int launch_sell_step(const sc_graph* g, const StepParams& p, cudaStream_t s, double* algo_bytes) {
  constexpr int W = Vec<T>::W;
  if (p.width % W) return fail(SC_ERR_ARG, "unsupported chunk width " + std::to_string(p.width));
  const int vpr = p.width / W;
  SellFn<T> k = pick_sell<T>(vpr, g->unit_weights, p.p2p != nullptr, p.mom_limbs != nullptr);
  if (!k) return fail(SC_ERR_ARG, "unsupported chunk width " + std::to_string(p.width));
  const int tr = sell_tile_rows(vpr);
  SellPlan* pl = nullptr;
  if (p.split_mode == 1) SC_TRY(sell_plan(g, vpr, p.row_begin, p.row_end, s, &pl, 0, p.split_col));
  else if (p.split_mode == 2) SC_TRY(sell_plan(g, vpr, p.row_begin, p.row_end, s, &pl, p.split_col, g->n_cols));
  else SC_TRY(sell_plan(g, vpr, p.row_begin, p.row_end, s, &pl));
  SellCfg cf = sell_config(tr, g->unit_weights, pl->max_tile);
  if (p.split_mode == 1 && cf.cap > 0) {   // no epilogue: no dense-row staging
    cf.dense = false;
    cf.smem = SellLayout(tr, cf.cap, g->unit_weights, cf.stages, false).total;
  }
  if (cf.cap <= 0) return fail(SC_ERR_STATE, "SELL tile exceeds the stage capacity");
  const int cap = cf.cap;
  const int smem = static_cast<int>(cf.smem);
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> occ_cache;
  static std::map<const void*, int> smem_attr;   // largest dynamic smem set per kernel
  int occ = 0;
  {
    std::lock_guard<std::mutex> lock(mu);
    int& attr = smem_attr[(const void*)k];
    if (smem > attr) {   // the attribute only grows: plans of one kernel differ in their smem
      SC_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      attr = smem;
    }
    auto it = occ_cache.find({(const void*)k, smem});
    if (it == occ_cache.end()) {
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kThreads, smem) != cudaSuccess || occ < 1) occ = 1;
      occ_cache[{(const void*)k, smem}] = occ;
    } else {
      occ = it->second;
    }
  }
  const int64_t rows = p.row_end - p.row_begin;
  if (rows <= 0) return SC_OK;
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(pl->ntiles, (int64_t)g->num_sms * occ)));
  SellDev sd{};
  sd.tile_ptr = pl->tile_ptr.as<int64_t>();
  sd.meta = pl->meta.as<int4>();
  sd.idx = pl->idx.as<int32_t>();
  sd.val = g->unit_weights ? nullptr : pl->val.as<float>();
  sd.order = pl->order.as<int32_t>();
  sd.hub_chunk_ptr = pl->hub_chunk_ptr.as<int32_t>();
  if (pl->n_chunks > 0 && p.split_mode != 1) {
    // split rows first: one warp per chunk of a hub row's edges -> hubpart (all of the row's
    // columns, also under the split gather: its first launch leaves hub rows at 0)
    SC_TRY(pl->hubpart.ensure(sizeof(T) * (size_t)pl->n_chunks * p.width));
    sd.hubpart = pl->hubpart.ptr;
    HubFn<T> hk = pick_hub<T>(vpr, g->unit_weights);
    const int hgrid = (int)std::min<int64_t>((pl->n_chunks + 7) / 8, (int64_t)g->num_sms * env_int_s("SC_HUB_BPS", 16));
    hk<<<hgrid, 256, 0, s>>>(pl->chunks.as<HubChunk>(), pl->n_chunks, g->col_idx.as<int32_t>(),
                             g->unit_weights ? nullptr : g->values.as<float>(), p, static_cast<T*>(pl->hubpart.ptr));
    SC_CUDA_TRY(cudaGetLastError());
  }
  const T* strength = sizeof(T) == 4 ? reinterpret_cast<const T*>(g->strength32.ptr)
                                     : reinterpret_cast<const T*>(g->strength64.ptr);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  SC_CUDA_TRY(cudaLaunchKernelEx(&cfg, k, sd, strength, p, cap, cf.packed()));
  if (algo_bytes) {
    // algorithmic bytes of the step: the CSR share of this chunk (row
    // pointers + column indices [+ weights], not the padding) + dense operands touched once
    const double csr = (double)rows * 8.0 + (double)g->nnz * (g->unit_weights ? 4.0 : 8.0) * rows / g->n_rows;
    const double dense_rows = (1.0 + (p.tprev ? 1.0 : 0.0) + (p.tnext ? 1.0 : 0.0) +
                               (p.y_mode == 2 ? 2.0 : (p.y_mode == 1 ? 1.0 : 0.0)));
    const double frac = (double)p.width / (p.total_width > 0 ? p.total_width : p.width);
    *algo_bytes = csr * frac + dense_rows * (double)rows * p.width * sizeof(T);
  }
  return SC_OK;
}
template <typename T>
int launch_step_any(const sc_graph* g, StepParams p, cudaStream_t s) {
  // With the fused exchange the SELL kernel pays register spills in its epilogue; measured per
  // rank (tools/grid_emulate.py, profiles/r02_grid_emulate_c4_sell.txt): 32-column chunks
  // equal or faster than the CSR kernel (c3, 8 ranks 21.9 vs 21.7 ms, 4 ranks 33.9 vs 35.2),
  // 48-column chunks 12-13 % slower (c4, 4 and 8 ranks) -- wider exchange chunks stay on CSR
  bool ok = false;
  const bool p2p_wide = p.p2p && (sizeof(T) != 4 || (p.width > 32 && !env_int_s("SC_P2P_SELL_WIDE", 0)));
  if (sell_enabled() && !p2p_wide) SC_TRY(sell_usable<T>(g, p.width, p.row_begin, p.row_end, s, &ok));
  if (!ok) return launch_step<T>(g, p, s);
  p.tile_ctr = dyn_tiles_on() ? next_tile_ctr(g, s) : nullptr;
  // the bench's per-launch events (sc_profile_begin), as launch_step records them
  cudaEvent_t e0 = nullptr;
  prof_launch_begin(s, &e0);
  double ab = 0.0;
  SC_TRY(launch_sell_step<T>(g, p, s, e0 ? &ab : nullptr));
  prof_launch_end(s, e0, ab, 1);
  return SC_OK;
}
template int launch_step_any<float>(const sc_graph*, StepParams, cudaStream_t);
template int launch_step_any<double>(const sc_graph*, StepParams, cudaStream_t);

template int launch_sell_step<float>(const sc_graph*, const StepParams&, cudaStream_t, double*);
template int launch_sell_step<double>(const sc_graph*, const StepParams&, cudaStream_t, double*);

}  // namespace sc
