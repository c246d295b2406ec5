// Fused Chebyshev recurrence step (CSR SpMM + three-term update + coefficient
// accumulation) and the drivers that run the whole filter.
//
// PAPER.md §2.4 Eq. (3) (lines 135-147): F^m_h x = sum_l alpha_l L^l x "only
// requires matrix-vector multiplication", realised (R1) as the
// Chebyshev three-term recurrence on L~ = (2/lambda_max) L - I:
//     T_0 = X,  T_1 = L~ X,  T_{j+1} = 2 L~ T_j - T_{j-1},   Y = sum_j d_j T_j.
// One launch = one recurrence step over all rows of one column chunk:
//     T_{s+1}[i] = a (s_i T_s[i] - sum_k W_ik T_s[k]) + b_cur T_s[i] + b_prev T_{s-1}[i]
//     Y[i]      (=|+=) cy_prev T_{s-1}[i] + cy_cur T_s[i] + cy_next T_{s+1}[i]
// with (a, b_cur, b_prev) = (2/lmax, -1, 0) at s = 0 and (4/lmax, -2, -1) after.
//
// Mapping: SW lanes per row, each lane owns one 16-byte
// vector of the row chunk (float4 / double2); a warp covers 32/SW rows.  The
// lanes of a row cooperatively load EB column indices per batch, broadcast them
// by warp shuffles and issue EB independent 16-byte gathers of T_s rows before
// consuming any (memory-level parallelism for the latency-bound gathers).
// Y is touched once every three steps (it needs T_{s-1}, T_s, T_{s+1}, which the
// step already holds in registers), so the fused step streams ~3.67 dense
// blocks instead of 5.
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>

#include "sc_internal.cuh"
#include "sc_ptx.cuh"

namespace sc {
namespace {

// ---------------------------------------------------------------------------
// The fused step kernel.
//
// Persistent CTAs (grid = SMs x resident CTAs) walk row tiles of TR = NC * (32/VPR)
// rows (tile t = blockIdx.x + i * gridDim.x).  Warp NC is the producer: for each
// tile it bulk-copies (cp.async.bulk, the TMA engine) the tile's row_ptr and
// col_idx (+ values) segments into an S-stage shared-memory ring guarded by
// full/empty mbarriers; lane j of the producer prefetches the CSR bounds of tile
// i+j, so one DRAM round trip serves 32 tiles.  Consumer warp c owns rows
// [r0 + c*RPW, r0 + (c+1)*RPW) of the tile, SW = VPR lanes per row, one 16-byte
// vector (float4 / double2) per lane, so every gathered row of T_s is read as
// VPR*16 contiguous bytes.  The own row, T_{s-1} and Y rows go to shared memory
// with cp.async (LDGSTS) -- no registers held across the gather loop.  Column
// indices are read from the staged segment (LDS); each gather address is one
// IMAD.WIDE.U32 off a per-lane base; a rolling window keeps EB independent
// 16-byte gathers in flight per lane.  Streaming operands carry an L2 evict-first
// policy so the gathered block T_s stays in L2.  A tile whose column segment
// exceeds the stage capacity reads col/values from global memory directly.
//
// MOMENTS (fp64): per-CTA partial sums of <T_s,T_s>, <T_{s+1},T_s>, <T_{s+1},T_{s+1}>.
// ---------------------------------------------------------------------------
// build-time tuning (native_build.py --defs)
#ifndef SC_NC
#define SC_NC 16          // consumer warps per CTA
#endif
#ifndef SC_MIN_CTAS
#define SC_MIN_CTAS 2     // resident CTAs per SM the register budget is sized for
#endif
#ifndef SC_EB_F32
#define SC_EB_F32 6       // gathers in flight per lane (fp32)
#endif
#ifndef SC_EB_F32W
#define SC_EB_F32W 5      // fp32, weighted graphs (6 spills: 168.7 vs 163.1 ms, c3 pattern with weights)
#endif
#ifndef SC_EB_F64
#define SC_EB_F64 5       // gathers in flight per lane (fp64; measured 4/5/6: 230/219/220 ms, c3 fp64 pass)
#endif
#ifndef SC_EB_F64_W
#define SC_EB_F64_W 4     // fp64, weighted graphs (5 spills)
#endif
#ifndef SC_EB_F64_MOM
#define SC_EB_F64_MOM 5   // fp64 with moments (per-tile warp-reduced partials, no spills: lambda_k on
                          // c3 126 / 121 / 170 ms for EB 4 / 5 / 6)
#endif
constexpr int kNC = SC_NC;
constexpr int kThreads = (kNC + 1) * 32;   // + one producer warp
#ifndef SC_NSTAGES
#define SC_NSTAGES 3      // CSR ring stages (4: 116.2 vs 115.0-115.6 ms on c3; the header fits 4)
#endif
constexpr int kMaxStages = SC_NSTAGES;
static_assert(kMaxStages <= 4, "barrier + TileMeta header holds at most 4 stages");

struct TileMeta {
  int64_t r0, r1;      // rows [r0, r1)
  int64_t rpa;         // first row_ptr index staged (r0 rounded down to even)
  int64_t ca;          // first col index staged (row_ptr[r0] rounded down to a multiple of 4)
  int32_t overflow;    // 1: the tile's col segment did not fit, read from global
  int32_t tile;        // tile index (dynamic scheduling); r0 < 0 marks the end
};

__host__ __device__ constexpr int tile_rows(int vpr) { return kNC * (32 / vpr); }

struct SmemLayout {
  int cap;          // col entries per stage
  int trp;          // row_ptr entries per stage
  int stages;
  size_t stage_bytes, rp_off, ord_off, col_off, val_off, dense_off, red_off, total;
  __host__ __device__ SmemLayout(int tr, int cap_, bool unit, int nst) {
    cap = cap_;
    stages = nst;
    trp = (tr + 4 + 1) & ~1;
    rp_off = 0;
    ord_off = (size_t)trp * 8;
    col_off = ord_off + (((size_t)tr * 2 + 15) & ~(size_t)15);
    val_off = col_off + (size_t)cap * 4;
    stage_bytes = val_off + (unit ? 0 : (size_t)cap * 4);
    stage_bytes = (stage_bytes + 127) & ~(size_t)127;
    dense_off = 256 + (size_t)stages * stage_bytes;
    red_off = dense_off + (size_t)kNC * 3 * 32 * 16;
    total = red_off + kNC * 3 * sizeof(double);
  }
};

template <typename T, int VPR, int EB, bool UNIT, bool MOMENTS>
__global__ void __launch_bounds__(kThreads, SC_MIN_CTAS)
cheb_step_kernel(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                 const float* __restrict__ val, const T* __restrict__ strength,
                 const uint16_t* __restrict__ order, StepParams p, int cap, int nstages) {
  constexpr int W = Vec<T>::W;
  constexpr int SW = VPR;          // lanes per row (one 16-byte vector each)
  constexpr int RPW = 32 / SW;     // rows per warp (lanes >= RPW*SW idle when SW does not divide 32)
  constexpr int TR = tile_rows(VPR);
  static_assert(VPR >= 1 && VPR <= 32, "VPR in [1, 32]");

  extern __shared__ __align__(128) unsigned char smem[];
  const SmemLayout lay(TR, cap, UNIT, nstages);
  const int S = nstages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + kMaxStages;
  TileMeta* meta = reinterpret_cast<TileMeta*>(smem + 64);
  unsigned char* stages = smem + 256;
  unsigned char* dense = smem + lay.dense_off;   // [kNC][3][32] x 16 bytes: own, prev, Y rows
  double* red = reinterpret_cast<double*>(smem + lay.red_off);

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

  // programmatic dependent launch: the next step's CTAs may become resident as this grid's
  // CTAs retire (its producer warps start staging CSR tiles, which no step writes); every
  // consumer waits for this whole grid (griddepcontrol.wait) before touching T, Y or the peers
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const uint64_t pol_stream = policy_evict_first();
  const unsigned own_c = p.l2pol & 3u, next_c = (p.l2pol >> 2) & 3u, prev_c = (p.l2pol >> 4) & 3u;
  const uint64_t pol_own = own_c == 0 ? pol_stream : (own_c == 1 ? policy_evict_normal() : policy_evict_last());
  const uint64_t pol_prev = prev_c == 0 ? pol_stream : policy_evict_normal();
  const uint64_t pol_next = next_c == 1 ? pol_stream : (next_c == 2 ? policy_evict_last() : policy_evict_normal());
#if SC_GATHER_HINT
  const uint64_t pol_gather = policy_gather();
#endif

  if (warp == kNC && p.tile_ctr) {
    // ------------------------------------------------- producer, dynamic schedule
    // tiles are taken one at a time from the launch's counter (the 3-stage ring hides the
    // atomic + bounds + bulk-copy chain); a stage with r0 = -1 tells the consumers to stop
    int i = 0;
    for (;; ++i) {
      const int s = i % S;
      if (lane == 0) {
        const unsigned tv = atomicAdd(p.tile_ctr, 1u);
        // the launch's last increment resets the slot (reusable without a host memset)
        if ((int64_t)tv == ntiles + gridDim.x - 1) atomicExch(p.tile_ctr, 0u);
        const int64_t t = tv;
        if (i >= S) mbar_wait(&empty[s], ((i / S) - 1) & 1);
        TileMeta& m = meta[s];
        if (t >= ntiles) {
          m.r0 = -1;
          mbar_arrive(&full[s]);
        } else {
          const int64_t r0 = p.row_begin + t * TR;
          const int64_t r1 = min(r0 + TR, p.row_end);
          const int64_t e0 = __ldg(row_ptr + r0), e1 = __ldg(row_ptr + r1);
          const int64_t rpa = r0 & ~int64_t(1);
          const int64_t nrp = ((r1 + 1 - rpa) + 1) & ~int64_t(1);
          const int64_t ca = e0 & ~int64_t(3);
          const int64_t ncol = ((e1 - ca) + 3) & ~int64_t(3);
          const int overflow = ncol > lay.cap;
          m.r0 = r0; m.r1 = r1; m.rpa = rpa; m.ca = ca; m.overflow = overflow; m.tile = (int32_t)t;
          unsigned char* st = stages + (size_t)s * lay.stage_bytes;
          uint32_t tx = (uint32_t)(nrp * 8) + (uint32_t)(TR * 2);
          const bool cp_col = !overflow && ncol > 0;
          if (cp_col) tx += (uint32_t)(ncol * 4 * (UNIT ? 1 : 2));
          mbar_arrive_expect_tx(&full[s], tx);
          bulk_g2s(st + lay.rp_off, row_ptr + rpa, (uint32_t)(nrp * 8), &full[s], pol_stream);
          bulk_g2s(st + lay.ord_off, order + t * TR, (uint32_t)(TR * 2), &full[s], pol_stream);
          if (cp_col) {
            bulk_g2s(st + lay.col_off, col + ca, (uint32_t)(ncol * 4), &full[s], pol_stream);
            if (!UNIT) bulk_g2s(st + lay.val_off, val + ca, (uint32_t)(ncol * 4), &full[s], pol_stream);
          }
        }
        i = t >= ntiles ? -i - 1 : i;   // (encode "done" for the warp)
      }
      i = __shfl_sync(FULL, i, 0);
      if (i < 0) { i = -i - 1; break; }
    }
    // drain: wait until the consumers released every real tile's stage still in use
    if (lane == 0)
      for (int j = max(0, i - S); j < i; ++j) mbar_wait(&empty[j % S], (j / S) & 1);
    return;
  }
  if (warp == kNC) {
    // ------------------------------------------------------------ producer
    int i = 0;
    for (int64_t tg = blockIdx.x; tg < ntiles; tg += (int64_t)gridDim.x * 32) {
      const int64_t tl = tg + (int64_t)lane * gridDim.x;
      int64_t b0 = 0, b1 = 0;
      if (tl < ntiles) {
        const int64_t r0 = p.row_begin + tl * TR;
        b0 = __ldg(row_ptr + r0);
        b1 = __ldg(row_ptr + min(r0 + TR, p.row_end));
      }
      const int64_t left = (ntiles - tg + gridDim.x - 1) / gridDim.x;
      const int cnt = left < 32 ? (int)left : 32;
      for (int j = 0; j < cnt; ++j, ++i) {
        const int64_t e0 = __shfl_sync(FULL, b0, j), e1 = __shfl_sync(FULL, b1, j);
        if (lane == 0) {
          const int s = i % S;
          if (i >= S) mbar_wait(&empty[s], ((i / S) - 1) & 1);
          const int64_t r0 = p.row_begin + (tg + (int64_t)j * gridDim.x) * TR;
          const int64_t r1 = min(r0 + TR, p.row_end);
          const int64_t rpa = r0 & ~int64_t(1);
          const int64_t nrp = ((r1 + 1 - rpa) + 1) & ~int64_t(1);
          const int64_t ca = e0 & ~int64_t(3);
          const int64_t ncol = ((e1 - ca) + 3) & ~int64_t(3);
          const int overflow = ncol > lay.cap;
          TileMeta& m = meta[s];
          m.r0 = r0; m.r1 = r1; m.rpa = rpa; m.ca = ca; m.overflow = overflow;
          unsigned char* st = stages + (size_t)s * lay.stage_bytes;
          uint32_t tx = (uint32_t)(nrp * 8) + (uint32_t)(TR * 2);
          const bool cp_col = !overflow && ncol > 0;
          if (cp_col) tx += (uint32_t)(ncol * 4 * (UNIT ? 1 : 2));
          mbar_arrive_expect_tx(&full[s], tx);
          bulk_g2s(st + lay.rp_off, row_ptr + rpa, (uint32_t)(nrp * 8), &full[s], pol_stream);
          bulk_g2s(st + lay.ord_off, order + (tg + (int64_t)j * gridDim.x) * TR, (uint32_t)(TR * 2), &full[s],
                   pol_stream);
          if (cp_col) {
            bulk_g2s(st + lay.col_off, col + ca, (uint32_t)(ncol * 4), &full[s], pol_stream);
            if (!UNIT) bulk_g2s(st + lay.val_off, val + ca, (uint32_t)(ncol * 4), &full[s], pol_stream);
          }
        }
      }
    }
    // drain: wait until the consumers released every stage still in use
    if (lane == 0)
      for (int j = max(0, i - S); j < i; ++j) mbar_wait(&empty[j % S], (j / S) & 1);
    return;
  }

  // -------------------------------------------------------------- consumers
  asm volatile("griddepcontrol.wait;" ::: "memory");   // the previous step has completed
  const int sub = lane / SW;
  const int sl = lane % SW;
  const int c = sl * W;   // first column of this lane's vector
  const T* tprev = static_cast<const T*>(p.tprev);   // may alias tnext (same row, read before write)
  const T* __restrict__ tcur = static_cast<const T*>(p.tcur);
  T* tnext = static_cast<T*>(p.tnext);
  T* y = static_cast<T*>(p.y);
  // gather address of row k for this lane: gbase + k * ldb (one IMAD.WIDE.U32)
  const char* gbase = reinterpret_cast<const char*>(tcur + c);
  const uint32_t ldb = static_cast<uint32_t>(p.ld_cur * sizeof(T));
  T* d_own = reinterpret_cast<T*>(dense + ((size_t)(warp * 3 + 0) * 32 + lane) * 16);
  T* d_prv = reinterpret_cast<T*>(dense + ((size_t)(warp * 3 + 1) * 32 + lane) * 16);
  T* d_y = reinterpret_cast<T*>(dense + ((size_t)(warp * 3 + 2) * 32 + lane) * 16);
  // MOMENTS: each tile's contributions are warp-reduced and added to this warp's slots of
  // `red` in tile order (deterministic), so no accumulator stays live across the gathers
  if (MOMENTS && lane < 3) red[warp * 3 + lane] = 0.0;

  int i = 0;
  const bool dyn = p.tile_ctr != nullptr;
  for (int64_t t = blockIdx.x; dyn || t < ntiles; t += gridDim.x, ++i) {
    const int s = i % S;
    mbar_wait(&full[s], (i / S) & 1);
    const TileMeta m = meta[s];
    if (dyn) {
      if (m.r0 < 0) break;   // the producer ran out of tiles
      t = m.tile;
    }
    const unsigned char* st = stages + (size_t)s * lay.stage_bytes;
    const int64_t* rps = reinterpret_cast<const int64_t*>(st + lay.rp_off);

    // rows of the tile in ascending-degree order; this warp takes one block of RPW
    // consecutive ranks (similar degrees -> little padding to the warp's longest row),
    // the block index rotating with the tile so every warp sees every degree class
    const uint16_t* ord = reinterpret_cast<const uint16_t*>(st + lay.ord_off);
    const int rank = ((warp + static_cast<int>(t % kNC)) % kNC) * RPW + sub;
    const bool valid = sub < RPW && rank < static_cast<int>(m.r1 - m.r0);
    const int64_t row = m.r0 + (valid ? ord[rank] : 0);
    int deg = 0;
    int64_t b = 0;
    double m_cc = 0.0, m_nc = 0.0, m_nn = 0.0;   // (MOMENTS) this tile's contributions
    T acc[W];
#pragma unroll
    for (int w = 0; w < W; ++w) acc[w] = T(0);
    if (valid) {
      b = rps[row - m.rpa];
      deg = static_cast<int>(rps[row - m.rpa + 1] - b);
      cp_async16(d_own, tcur + row * p.ld_cur + c, pol_own);
      if (tprev) cp_async16(d_prv, tprev + row * p.ld_prev + c, pol_prev);
      if (p.y_mode == 2) cp_async16(d_y, y + row * p.ld_y + c, pol_stream);
    }
    int maxdeg = deg;   // over the warp's rows (an upper bound of each row's degree)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) maxdeg = max(maxdeg, __shfl_xor_sync(FULL, maxdeg, o));

    // Rolling window of EB gathers: slot e always holds the load of edge base+e; consuming it
    // (scoreboard wait on that load only) is immediately followed by issuing edge base+EB+e,
    // so EB independent 16-byte loads stay in flight per lane across the whole row.
    auto gather = [&](const int32_t* __restrict__ ci, const float* __restrict__ wi) {
      T g[EB][W];
      T wv[EB];
      auto issue = [&](int e, int pos) {
        const bool ok = pos < deg;
        const int k = ok ? ci[pos] : 0;
        if (!UNIT) wv[e] = ok ? static_cast<T>(wi[pos]) : T(0);
        if (ok) {
#if SC_GATHER_HINT
          Stream<T>::ld_hint(reinterpret_cast<const T*>(gbase + static_cast<uint64_t>(static_cast<uint32_t>(k)) * ldb),
                             g[e], pol_gather);
#else
          Vec<T>::ldg(reinterpret_cast<const T*>(gbase + static_cast<uint64_t>(static_cast<uint32_t>(k)) * ldb), g[e]);
#endif
        } else {
#pragma unroll
          for (int w = 0; w < W; ++w) g[e][w] = T(0);
        }
      };
#pragma unroll
      for (int e = 0; e < EB; ++e) issue(e, e);
      for (int base = 0; base < maxdeg; base += EB) {
#pragma unroll
        for (int e = 0; e < EB; ++e) {
#pragma unroll
          for (int w = 0; w < W; ++w) {
            if (UNIT) acc[w] += g[e][w];
            else acc[w] = fma(wv[e], g[e][w], acc[w]);
          }
          issue(e, base + EB + e);
        }
      }
    };
    if (!m.overflow) {
      // column indices (and weights) from the staged shared-memory segment
      gather(reinterpret_cast<const int32_t*>(st + lay.col_off) + (b - m.ca),
             reinterpret_cast<const float*>(st + lay.val_off) + (b - m.ca));
    } else {
      gather(col + b, UNIT ? nullptr : val + b);
    }
    // all lanes of this warp are done with stage s
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);

    if (valid) {
      asm volatile("cp.async.wait_all;" ::: "memory");
      T own[W], prv[W], yv[W];
      Vec<T>::ld(d_own, own);
      if (tprev) Vec<T>::ld(d_prv, prv);
      else {
#pragma unroll
        for (int w = 0; w < W; ++w) prv[w] = T(0);
      }
      if (p.y_mode == 2) Vec<T>::ld(d_y, yv);
      else {
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
      if (tnext) {   // T_{s+1} is gathered next step: normal L2 policy by default
        if (next_c == 0) Vec<T>::st(tnext + row * p.ld_next + c, tn);
        else Stream<T>::st(tnext + row * p.ld_next + c, tn, pol_next);
      }
      if (p.p2p && tnext && row >= p.p2p->row0) {
        // fused halo exchange: the peers that read this row get it straight into their halo
        // (NVLink stores from the epilogue, no pack / send / receive)
        const P2PDev* x = p.p2p;
        const int64_t e1 = x->sd_ptr[row + 1];
        for (int64_t e = x->sd_ptr[row]; e < e1; ++e) {
          const int q = x->sd_peer[e];
          T* dst = static_cast<T*>(x->peer_buf[p.p2p_next][q]) + (x->peer_nl[q] + x->sd_slot[e]) * p.ld_next + c;
          Vec<T>::st(dst, tn);
        }
      }
      if (p.y_mode) {
        const T cyp = static_cast<T>(p.cy_prev), cyc = static_cast<T>(p.cy_cur), cyn = static_cast<T>(p.cy_next);
#pragma unroll
        for (int w = 0; w < W; ++w) yv[w] += cyp * prv[w] + cyc * own[w] + cyn * tn[w];
        Stream<T>::st(y + row * p.ld_y + c, yv, pol_stream);
      }
      if (MOMENTS) {
#pragma unroll
        for (int w = 0; w < W; ++w) {
          const double o = own[w], n = tn[w];
          m_cc += o * o;
          m_nc += n * o;
          m_nn += n * n;
        }
      }
    }
    if (MOMENTS) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        m_cc += __shfl_xor_sync(FULL, m_cc, o);
        m_nc += __shfl_xor_sync(FULL, m_nc, o);
        m_nn += __shfl_xor_sync(FULL, m_nn, o);
      }
      if (lane == 0) {
        red[warp * 3 + 0] += m_cc;
        red[warp * 3 + 1] += m_nc;
        red[warp * 3 + 2] += m_nn;
      }
    }
  }

  if (p.p2p) {
    // publish completion to the peers: every consumer thread fences its (remote) stores,
    // the last CTA to finish writes p2p_signal into each peer's flag array (release)
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

  if (MOMENTS) {
    // deterministic CTA reduction over the consumer warps' slots (named barrier 1)
    asm volatile("bar.sync 1, %0;" ::"r"(kNC * 32) : "memory");
    if (threadIdx.x < 3) {
      double sum = 0.0;
      for (int w = 0; w < kNC; ++w) sum += red[w * 3 + threadIdx.x];
      p.part[blockIdx.x * 3 + threadIdx.x] = sum;
    }
  }
}

// Degree-sorted row order inside each tile: order[t*tr + rank] = local row index, ranks by
// (degree, index).  Built once per (graph, tile rows, row range) and cached on the graph.
__global__ void tile_order_kernel(const int64_t* __restrict__ row_ptr, int64_t row_begin, int64_t row_end, int tr,
                                  uint16_t* __restrict__ order) {
  extern __shared__ int degs[];
  const int64_t t = blockIdx.x;
  const int64_t r0 = row_begin + t * tr;
  const int cnt = static_cast<int>(min((int64_t)tr, row_end - r0));
  for (int i = threadIdx.x; i < tr; i += blockDim.x)
    degs[i] = i < cnt ? static_cast<int>(row_ptr[r0 + i + 1] - row_ptr[r0 + i]) : INT_MAX;
  __syncthreads();
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
    const int d = degs[i];
    int rank = 0;
    for (int j = 0; j < cnt; ++j) {
      const int dj = degs[j];
      rank += (dj < d) || (dj == d && j < i);
    }
    order[t * tr + rank] = static_cast<uint16_t>(i);
  }
  for (int i = cnt + threadIdx.x; i < tr; i += blockDim.x) order[t * tr + i] = 0;
}

// sum per-block moment partials of one launch in a fixed order
__global__ void reduce_partials_kernel(const double* __restrict__ part, int nblocks,
                                       double* __restrict__ out) {
  __shared__ double sh[3][256];
  for (int comp = 0; comp < 3; ++comp) {
    double s = 0.0;
    for (int b = threadIdx.x; b < nblocks; b += blockDim.x) s += part[b * 3 + comp];
    sh[comp][threadIdx.x] = s;
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    double s = 0.0;
    for (int t = 0; t < (int)blockDim.x; ++t) s += sh[threadIdx.x][t];
    out[threadIdx.x] = s;
  }
}

template <typename T>
__global__ void copy_cols_kernel(const T* __restrict__ src, int64_t lds, T* __restrict__ dst,
                                 int64_t ldd, int64_t n, int cols) {
  const int64_t total = n * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols;
    const int c = static_cast<int>(i % cols);
    dst[r * ldd + c] = src[r * lds + c];
  }
}

// ---------------------------------------------------------------------------
// launch profiler (sc_profile_begin / sc_profile_end): CUDA events around every
// fused-step launch on the launching stream, plus a count of all kernels the
// filter path launches.
// ---------------------------------------------------------------------------
struct Prof {
  bool on = false;
  int64_t launches = 0;        // every kernel launched by the filter path
  int64_t step_launches = 0;   // fused-step launches
  double algo_bytes = 0.0;     // algorithmic bytes of the timed step launches
  std::vector<cudaEvent_t> pool;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
  size_t used = 0;
  cudaEvent_t get() {
    if (used == pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      pool.push_back(e);
    }
    return pool[used++];
  }
};
Prof g_prof;

// ---------------------------------------------------------------------------
// tuning knobs (env SC_CHUNK, SC_L2_BUDGET_MB, SC_RESIDENT) -- see DESIGN.md
// ---------------------------------------------------------------------------
int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}

// SC_PERSIST_MB > 0 (experiment): reserve that much L2 for persisting lines and launch every
// step with an access-policy window over its gathered table
size_t g_persist_max_window = 0;
size_t persist_bytes() {
  static const size_t v = [] {
    const int mb = env_int("SC_PERSIST_MB", 0);
    if (mb <= 0) return (size_t)0;
    int dev = 0, maxp = 0, maxw = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev);
    cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, dev);
    const size_t want = std::min((size_t)mb << 20, (size_t)maxp);
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want);
    size_t got = 0;
    cudaDeviceGetLimit(&got, cudaLimitPersistingL2CacheSize);
    g_persist_max_window = (size_t)maxw;
    std::fprintf(stderr, "[sc] persisting L2: max %d B, window max %d B, set %zu B\n", maxp, maxw, got);
    return got;
  }();
  return v;
}
size_t persist_max_window() { return g_persist_max_window; }

// SC_L2_SETASIDE_MB > 0 (experiment): L2 set-aside for persisting (evict_last) lines, no window
void setaside_once() {
  static const bool done = [] {
    const int mb = env_int("SC_L2_SETASIDE_MB", 0);
    if (mb > 0) {
      int dev = 0, maxp = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev);
      cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, std::min((size_t)mb << 20, (size_t)maxp));
      size_t got = 0;
      cudaDeviceGetLimit(&got, cudaLimitPersistingL2CacheSize);
      std::fprintf(stderr, "[sc] L2 set-aside %zu B (max %d)\n", got, maxp);
    }
    return true;
  }();
  (void)done;
}

}  // namespace

// dynamic tile scheduling of the step kernel (env SC_DYN_TILES=0 disables)
bool dyn_tiles_on() {
  static const bool v = env_int("SC_DYN_TILES", 1) != 0;
  return v;
}
constexpr int kTileCtrRing = 1024;
unsigned* next_tile_ctr(const sc_graph* g, cudaStream_t s) {
  std::lock_guard<std::mutex> lock(g->tile_ctr_mu);
  if (!g->tile_ctr_ring.ptr) {
    if (g->tile_ctr_ring.ensure(sizeof(unsigned) * kTileCtrRing) != SC_OK) return nullptr;
    if (cudaMemsetAsync(g->tile_ctr_ring.ptr, 0, sizeof(unsigned) * kTileCtrRing, s) != cudaSuccess) return nullptr;
    if (cudaStreamSynchronize(s) != cudaSuccess) return nullptr;   // zeroed before any stream uses it
  }
  // every slot is reset to 0 by the last tile request of the launch that used it (the step
  // kernels' producers), so the ring needs no re-zeroing when it wraps; kTileCtrRing
  // launches in flight at once would be needed to reuse a slot early
  const int idx = static_cast<int>(g->tile_ctr_seq++ % kTileCtrRing);
  return g->tile_ctr_ring.as<unsigned>() + idx;
}

namespace {

// step launches with programmatic dependent launch (env SC_PDL=0 disables; measured neutral on
// configs[3]: 115.2 vs 115.3 ms per pass -- a ~290 us launch has little prologue to hide)
bool pdl_on() {
  static const bool v = env_int("SC_PDL", 1) != 0;
  return v;
}

template <typename T>
using KernelFn = void (*)(const int64_t*, const int32_t*, const float*, const T*, const uint16_t*, StepParams, int,
                          int);

// EBU / EBW: gathers in flight per lane for unit / weighted graphs (weights take registers)
template <typename T, int VPR, int EBU, int EBW, bool MOM>
KernelFn<T> pick_unit(bool unit) {
  if (unit) return cheb_step_kernel<T, VPR, EBU, true, MOM>;
  return cheb_step_kernel<T, VPR, EBW, false, MOM>;
}

template <typename T, int EBU, int EBW, bool MOM>
KernelFn<T> pick_vpr(int vpr, bool unit) {
  switch (vpr) {
    case 1: return pick_unit<T, 1, EBU, EBW, MOM>(unit);
    case 2: return pick_unit<T, 2, EBU, EBW, MOM>(unit);
    case 3: return pick_unit<T, 3, EBU, EBW, MOM>(unit);
    case 4: return pick_unit<T, 4, EBU, EBW, MOM>(unit);
    case 6: return pick_unit<T, 6, EBU, EBW, MOM>(unit);
    case 8: return pick_unit<T, 8, EBU, EBW, MOM>(unit);
    case 12: return pick_unit<T, 12, EBU, EBW, MOM>(unit);
    case 16: return pick_unit<T, 16, EBU, EBW, MOM>(unit);
    case 24: return pick_unit<T, 24, EBU, EBW, MOM>(unit);
    case 32: return pick_unit<T, 32, EBU, EBW, MOM>(unit);
    default: return nullptr;
  }
}

template <typename T>
KernelFn<T> pick_kernel(int width, bool unit, bool moments) {
  constexpr int W = Vec<T>::W;
  if (width % W) return nullptr;
  const int vpr = width / W;
  // SC_EB_* gathers of 16 bytes in flight per lane within the 56-register budget of 2 x
  // 544-thread CTAs per SM (the 128-byte-row unit-weight kernels the configs use do not spill;
  // the weighted fp32, moments and odd-width fp64 variants spill a few bytes)
  if (moments) {
    if constexpr (sizeof(T) == 8) return pick_vpr<T, SC_EB_F64_MOM, SC_EB_F64_MOM, true>(vpr, unit);
    return nullptr;   // moments are accumulated in fp64 only
  }
  if constexpr (sizeof(T) == 4) return pick_vpr<T, SC_EB_F32, SC_EB_F32W, false>(vpr, unit);
  else return pick_vpr<T, SC_EB_F64, SC_EB_F64_W, false>(vpr, unit);
}

template <typename T> const T* strength_of(const sc_graph* g);
template <> const float* strength_of<float>(const sc_graph* g) { return g->strength32.as<float>(); }
template <> const double* strength_of<double>(const sc_graph* g) { return g->strength64.as<double>(); }

// Pipeline depth and column-index capacity of one stage: 3 stages with room for
// ~48 entries per tile row (average degree <= ~40 keeps nearly every tile on the
// staged path), capped so the CTA stays under ~100 KB of shared memory (2 CTAs per
// SM).  Tiles whose segment exceeds the capacity read their columns from global
// memory (correct, slower).
void stage_plan(int tr, bool unit, int* cap, int* nstages) {
  const int ns = kMaxStages;
  const int per_entry = unit ? 4 : 8;
  const int budget = 100 * 1024 - 256 - kNC * 3 * 32 * 16 - kNC * 3 * 8;
  const int per_stage = budget / ns - (tr + 6) * 8 - tr * 2 - 144;
  int c = std::min(tr * 48, per_stage / per_entry);
  *cap = std::max(64, c & ~3);
  *nstages = ns;
}

template <typename T>
int launch_step_impl(const sc_graph* g, const StepParams& p, cudaStream_t s, bool moments,
                     int* grid_out) {
  constexpr int W = Vec<T>::W;
  KernelFn<T> k = pick_kernel<T>(p.width, g->unit_weights, moments);
  if (!k) return fail(SC_ERR_ARG, "unsupported chunk width " + std::to_string(p.width));
  const int vpr = p.width / W;
  const int tr = tile_rows(vpr);
  int cap = 0, nst = 0;
  stage_plan(tr, g->unit_weights, &cap, &nst);
  const SmemLayout lay(tr, cap, g->unit_weights, nst);
  const int smem = static_cast<int>(lay.total);
  // per (kernel, smem size) launch configuration, resolved once per process
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> occ_cache;
  int occ = 0;
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = occ_cache.find({(const void*)k, smem});
    if (it == occ_cache.end()) {
      SC_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kThreads, smem) != cudaSuccess || occ < 1) occ = 1;
      occ_cache[{(const void*)k, smem}] = occ;
    } else {
      occ = it->second;
    }
  }
  const int64_t rows = p.row_end - p.row_begin;
  const int64_t ntiles = (rows + tr - 1) / tr;
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)g->num_sms * occ)));
  if (grid_out) *grid_out = grid;
  if (rows <= 0) return SC_OK;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (g_prof.on) {
    e0 = g_prof.get();
    e1 = g_prof.get();
    cudaEventRecord(e0, s);
  }
  const uint16_t* order = tile_order(g, tr, p.row_begin, p.row_end, s);
  if (!order) return fail(SC_ERR_NOMEM, "tile order allocation failed");
  StepParams q = p;
  // moments: static round-robin tiles, so each CTA's partial sums cover the same tiles in the
  // same order on every run (deterministic moments -> deterministic lambda_k)
  q.tile_ctr = (dyn_tiles_on() && !moments) ? next_tile_ctr(g, s) : nullptr;
  q.l2pol = static_cast<unsigned>(env_int("SC_L2POL", 0));
  setaside_once();
  const size_t persist = persist_bytes();
  if (persist) {
    // experiment (SC_PERSIST_MB): an L2 persisting window over the gathered table T_s
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeAccessPolicyWindow;
    const size_t tbytes = (size_t)g->n_cols * p.ld_cur * sizeof(T);
    at[0].val.accessPolicyWindow.base_ptr = const_cast<void*>(p.tcur);
    at[0].val.accessPolicyWindow.num_bytes = std::min(tbytes, persist_max_window());
    at[0].val.accessPolicyWindow.hitRatio = (float)std::min(1.0, (double)persist / (double)tbytes);
    at[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    at[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    SC_CUDA_TRY(cudaLaunchKernelEx(&cfg, k, g->row_ptr.as<int64_t>(), g->col_idx.as<int32_t>(),
                                   g->unit_weights ? nullptr : g->values.as<float>(), strength_of<T>(g), order, q, cap,
                                   nst));
  } else if (pdl_on()) {
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
    SC_CUDA_TRY(cudaLaunchKernelEx(&cfg, k, g->row_ptr.as<int64_t>(), g->col_idx.as<int32_t>(),
                                   g->unit_weights ? nullptr : g->values.as<float>(), strength_of<T>(g), order, q, cap,
                                   nst));
  } else {
    k<<<grid, kThreads, smem, s>>>(g->row_ptr.as<int64_t>(), g->col_idx.as<int32_t>(),
                                   g->unit_weights ? nullptr : g->values.as<float>(), strength_of<T>(g), order, q, cap,
                                   nst);
  }
  SC_CUDA_TRY(cudaGetLastError());
  if (g_prof.on) {
    cudaEventRecord(e1, s);
    g_prof.ev.emplace_back(e0, e1);
    g_prof.launches += 1;
    g_prof.step_launches += 1;
    // algorithmic bytes: CSR share of this chunk + dense operands touched once
    const double csr = (double)rows * 8.0 + (double)g->nnz * (g->unit_weights ? 4.0 : 8.0) * rows / g->n_rows;
    const double dense_rows = (1.0 + (p.tprev ? 1.0 : 0.0) + (p.tnext ? 1.0 : 0.0) +
                               (p.y_mode == 2 ? 2.0 : (p.y_mode == 1 ? 1.0 : 0.0)));
    const double frac = (double)p.width / (p.total_width > 0 ? p.total_width : p.width);
    g_prof.algo_bytes += csr * frac + dense_rows * (double)rows * p.width * sizeof(T);
  }
  return SC_OK;
}

// Split R columns into chunks of supported widths, each <= cw.
// Row widths (in 16-byte vectors) the kernels are instantiated for.
constexpr int kVprSet[] = {32, 24, 16, 12, 8, 6, 4, 3, 2, 1};

// Split R columns (a multiple of the vector width) into chunks of supported widths, each
// at most cw.
template <typename T>
std::vector<int> chunk_plan(int R, int64_t n_cols) {
  constexpr int W = Vec<T>::W;
  const int maxv = 32;   // one warp per row
  int cv = env_int("SC_CHUNK", 0) / W;
  if (cv <= 0) {
    // Keep the gathered chunk of T_s L2-resident: the widest supported row whose N x w block
    // fits the budget.  If that would take rows narrower than 128 bytes, the block cannot be
    // L2-resident at a useful row size anyway: use 256-byte rows (large DRAM requests, half
    // the CSR re-reads of 128-byte rows; measured on configs[4]: 64 + 32 columns 3.88 s,
    // one 96-column chunk 4.09 s, one padded 128-column chunk 5.09 s per pass).
    const double budget = env_int("SC_L2_BUDGET_MB", 128) * 1048576.0;
    cv = 1;
    for (int v : kVprSet)
      if ((double)n_cols * v * 16 <= budget) { cv = v; break; }
    if (cv * 16 < 128) cv = 16;
  }
  cv = std::max(1, std::min(cv, maxv));
  std::vector<int> out;
  int rem = R / W;
  while (rem > 0) {
    int v = 1;
    for (int c : kVprSet)
      if (c <= rem && c <= cv) { v = c; break; }
    out.push_back(v * W);
    rem -= v;
  }
  return out;
}

}  // namespace

const uint16_t* tile_order(const sc_graph* g, int tr, int64_t row_begin, int64_t row_end, cudaStream_t s) {
  std::lock_guard<std::mutex> lock(g->tile_orders_mu);
  auto key = std::make_tuple(tr, row_begin, row_end);
  auto it = g->tile_orders.find(key);
  if (it != g->tile_orders.end()) return it->second->as<uint16_t>();
  const int64_t ntiles = (row_end - row_begin + tr - 1) / tr;
  auto buf = std::make_unique<DevBuf>();
  if (buf->ensure(sizeof(uint16_t) * (size_t)std::max<int64_t>(1, ntiles) * tr) != SC_OK) return nullptr;
  if (ntiles > 0) {
    tile_order_kernel<<<(unsigned)ntiles, 256, sizeof(int) * tr, s>>>(g->row_ptr.as<int64_t>(), row_begin, row_end, tr,
                                                                     buf->as<uint16_t>());
    if (cudaGetLastError() != cudaSuccess) return nullptr;
  }
  const uint16_t* out = buf->as<uint16_t>();
  g->tile_orders[key] = std::move(buf);
  return out;
}

void prof_launch_begin(cudaStream_t s, cudaEvent_t* e0) {
  *e0 = nullptr;
  if (!g_prof.on) return;
  *e0 = g_prof.get();
  cudaEventRecord(*e0, s);
}

void prof_launch_end(cudaStream_t s, cudaEvent_t e0, double algo_bytes, int steps) {
  if (!g_prof.on || !e0) return;
  cudaEvent_t e1 = g_prof.get();
  cudaEventRecord(e1, s);
  g_prof.ev.emplace_back(e0, e1);
  g_prof.launches += 1;
  g_prof.step_launches += steps;
  g_prof.algo_bytes += algo_bytes;
}

template <typename T>
std::vector<int> chunk_widths(int R, int64_t n_cols) {
  return chunk_plan<T>(R, n_cols);
}
template std::vector<int> chunk_widths<float>(int, int64_t);
template std::vector<int> chunk_widths<double>(int, int64_t);

void profile_begin() {
  g_prof.on = true;
  g_prof.launches = 0;
  g_prof.step_launches = 0;
  g_prof.algo_bytes = 0.0;
  g_prof.ev.clear();
  g_prof.used = 0;
}

int profile_end(int64_t* launches, int64_t* step_launches, double* step_ms, double* algo_bytes) {
  g_prof.on = false;
  double tot = 0.0;
  for (auto& pr : g_prof.ev) {
    SC_CUDA_TRY(cudaEventSynchronize(pr.second));
    float ms = 0.f;
    SC_CUDA_TRY(cudaEventElapsedTime(&ms, pr.first, pr.second));
    tot += ms;
  }
  if (launches) *launches = g_prof.launches;
  if (step_launches) *step_launches = g_prof.step_launches;
  if (step_ms) *step_ms = tot;
  if (algo_bytes) *algo_bytes = g_prof.algo_bytes;
  g_prof.ev.clear();
  g_prof.used = 0;
  return SC_OK;
}

template <typename T>
int launch_step(const sc_graph* g, const StepParams& p, cudaStream_t s) {
  return launch_step_impl<T>(g, p, s, false, nullptr);
}
template int launch_step<float>(const sc_graph*, const StepParams&, cudaStream_t);
template int launch_step<double>(const sc_graph*, const StepParams&, cudaStream_t);

int launch_moments_step(const sc_graph* g, const StepParams& p, cudaStream_t s, int* grid) {
  return launch_step_impl<double>(g, p, s, true, grid);
}

int reduce_moment_partials(const double* part, int grid, double* out, cudaStream_t s) {
  reduce_partials_kernel<<<1, 256, 0, s>>>(part, grid, out);
  SC_CUDA_TRY(cudaGetLastError());
  return SC_OK;
}

// ---------------------------------------------------------------------------
// whole filter on device buffers
// ---------------------------------------------------------------------------
// edges (i, j) with |i - j| < band (the ordering's locality), one pass over the CSR
__global__ void local_edges_kernel(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col, int64_t n,
                                   int64_t band, unsigned long long* __restrict__ out) {
  unsigned long long c = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
      const int64_t d = (int64_t)col[e] - i;
      c += (d < band && d > -band) ? 1ull : 0ull;
    }
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, c);
}

// Chunk width from the graph's structure (round 2).  When the L2-budget rule of chunk_plan picks
// 32-column chunks (the 32-column gathered table fits the budget, a 64-column one does not:
// graphs of ~0.5-1M nodes) and the block has >= 64 columns, 64-column chunks are used instead
// when the gathers concentrate -- power-law degrees (max degree > 8x the mean, the SELL plan's
// skew test) or a local ordering (>= half of the edges within n/64 rows) -- so that the hot rows
// of the 256 MB table stay in L2 and the per-row work halves.  Measured (ms per p = 200 pass,
// R = 64, one box): Chung-Lu 119.6 vs 125.3, RCM-ordered kNN 89.8 vs 99.7, but the uniform
// random configs[3] 110.4 vs 103.5 (`profiles/r02_tune.txt`, `r02_c3_64.txt`).  A structural
// rule, not a timing, so a graph always gets the same width (hub rows' sums depend on it in the
// last bits, R15).  Cached per graph; env SC_CHUNK_WIDE = 0 / 1 forces it off / on.
int wide_chunks(sc_graph* g, cudaStream_t s, bool* wide) {
  *wide = false;
  const int forced = env_int("SC_CHUNK_WIDE", -1);
  if (forced >= 0) {
    *wide = forced != 0;
    return SC_OK;
  }
  std::lock_guard<std::mutex> lock(g->chunk_tuned_mu);   // concurrent filter calls on one graph
  auto it = g->chunk_tuned.find(std::make_pair(0, 0));
  if (it != g->chunk_tuned.end()) {
    *wide = it->second != 0;
    return SC_OK;
  }
  const double mean = (double)g->nnz / std::max<int64_t>(1, g->n_rows);
  bool w = (double)max_row_degree(g, 0, g->n_rows, s) > 8.0 * std::max(1.0, mean);
  if (!w && g->nnz > 0) {
    DevBuf b;
    SC_TRY(b.ensure(sizeof(unsigned long long)));
    unsigned long long h = 0;
    SC_CUDA_TRY(cudaMemsetAsync(b.ptr, 0, sizeof(h), s));
    local_edges_kernel<<<g->num_sms * 8, 256, 0, s>>>(g->row_ptr.as<int64_t>(), g->col_idx.as<int32_t>(), g->n_rows,
                                                       std::max<int64_t>(1, g->n_rows / 64),
                                                       b.as<unsigned long long>());
    SC_CUDA_TRY(cudaGetLastError());
    SC_CUDA_TRY(cudaMemcpyAsync(&h, b.ptr, sizeof(h), cudaMemcpyDeviceToHost, s));
    SC_CUDA_TRY(cudaStreamSynchronize(s));
    w = 2 * h >= (unsigned long long)g->nnz;
  }
  g->chunk_tuned[std::make_pair(0, 0)] = w ? 1 : 0;
  *wide = w;
  return SC_OK;
}

template <typename T>
int tuned_chunk_plan(sc_graph* g, int Rp, cudaStream_t s, std::vector<int>* out) {
  *out = chunk_plan<T>(Rp, g->n_cols);
  if (sizeof(T) != 4 || Rp < 64 || env_int("SC_CHUNK", 0) > 0 || !sell_enabled() || out->empty() ||
      (*out)[0] != 32 || g->n_cols != g->n_rows)
    return SC_OK;
  bool wide = false;
  SC_TRY(wide_chunks(g, s, &wide));
  if (!wide) return SC_OK;
  std::vector<int> c;
  int rem = Rp;
  while (rem >= 64) {
    c.push_back(64);
    rem -= 64;
  }
  if (rem > 0) {
    const std::vector<int> tail = chunk_plan<T>(rem, g->n_cols);
    c.insert(c.end(), tail.begin(), tail.end());
  }
  *out = c;
  return SC_OK;
}

template <typename T>
int filter_apply(sc_graph* g, const double* d, int order, double lambda_max, int R, const T* X,
                 T* Y, cudaStream_t s) {
  constexpr int W = Vec<T>::W;
  const int64_t n = g->n_rows;
  // operate on a vector-aligned layout; pad odd widths / misaligned pointers.  A width that
  // is not a single supported chunk (e.g. R = 24 -> 16 + 8) is padded up to the next power
  // of two when that still fits one L2-sized chunk: one launch per step instead of several
  // (small graphs are launch-bound).
  int Rp = (R + W - 1) / W * W;
  {
    // smallest supported width >= Rp
    int pv = 32;
    for (int v : kVprSet)
      if (v * W >= Rp) pv = v;
    const int p2 = pv * W;
    const std::vector<int> one = chunk_plan<T>(p2, g->n_cols);
    const bool resident = (double)g->n_cols * p2 * sizeof(T) <= env_int("SC_L2_BUDGET_MB", 128) * 1048576.0;
    if (p2 > Rp && resident && one.size() == 1 && chunk_plan<T>(Rp, g->n_cols).size() > 1) Rp = p2;
  }
  const bool aligned = (Rp == R) && ((uintptr_t)X % 16 == 0) && ((uintptr_t)Y % 16 == 0);
  const T* Xw = X;
  T* Yw = Y;
  if (!aligned) {
    SC_TRY(g->ws_sig.ensure((size_t)2 * n * Rp * sizeof(T)));
    T* xp = g->ws_sig.as<T>();
    T* yp = xp + (size_t)n * Rp;
    SC_CUDA_TRY(cudaMemsetAsync(xp, 0, (size_t)n * Rp * sizeof(T), s));
    copy_cols_kernel<T><<<g->num_sms * 8, 256, 0, s>>>(X, R, xp, Rp, n, R);
    SC_CUDA_TRY(cudaGetLastError());
    if (g_prof.on) g_prof.launches += 1;
    Xw = xp;
    Yw = yp;
  }
  std::vector<int> chunks;
  SC_TRY(tuned_chunk_plan<T>(g, Rp, s, &chunks));
  int cwmax = 0;
  for (int w : chunks) cwmax = std::max(cwmax, w);
  // + one row: the all-zero row n_cols that the SELL padding gathers
  SC_TRY(g->ws_a.ensure((size_t)(g->n_cols + 1) * cwmax * sizeof(T)));
  SC_TRY(g->ws_b.ensure((size_t)(g->n_cols + 1) * cwmax * sizeof(T)));

  int col0 = 0;
  for (int w : chunks) {
    T* bufs[2] = {g->ws_b.as<T>(), g->ws_a.as<T>()};   // T_j lives in bufs[j & 1]
    const T* Xc = Xw + col0;
    T* Yc = Yw + col0;
    // small graphs: one cooperative launch for all steps, CSR resident in shared memory
    if (env_int("SC_RESIDENT", 1)) {
      bool ok = false;
      SC_TRY(resident_filter<T>(g, d, order, lambda_max, w, Xc, Rp, Yc, Rp, bufs[0], bufs[1], s, &ok));
      if (ok) {
        col0 += w;
        continue;
      }
    }
    bool use_sell = false;
    int64_t split_col = 0;
    if (sell_enabled()) {
      split_col = sell_split_col(g, w, sizeof(T));
      if (split_col > 0) SC_TRY(sell_usable<T>(g, w, 0, n, s, &use_sell, split_col));
      if (!use_sell) {
        split_col = 0;
        SC_TRY(sell_usable<T>(g, w, 0, n, s, &use_sell));
      }
    }
    if (split_col > 0) SC_TRY(g->ws_split.ensure(sizeof(T) * (size_t)n * w));
    if (use_sell) {
      // SELL path: T_0 = the X chunk copied into bufs[0] (row stride w), zero row n_cols in
      // both buffers (the sentinel of the padded slices)
      SC_CUDA_TRY(cudaMemsetAsync(bufs[0] + (size_t)g->n_cols * w, 0, sizeof(T) * w, s));
      SC_CUDA_TRY(cudaMemsetAsync(bufs[1] + (size_t)g->n_cols * w, 0, sizeof(T) * w, s));
      copy_cols_kernel<T><<<g->num_sms * 8, 256, 0, s>>>(Xc, Rp, bufs[0], w, n, w);
      SC_CUDA_TRY(cudaGetLastError());
      if (g_prof.on) g_prof.launches += 1;
      int added = -1;
      for (int st = 0; st < order; ++st) {
        StepParams p{};
        p.row_begin = 0;
        p.row_end = n;
        p.width = w;
        p.total_width = Rp;
        p.tcur = bufs[st & 1];
        p.ld_cur = w;
        p.tprev = st == 0 ? nullptr : (const void*)bufs[(st - 1) & 1];
        p.ld_prev = w;
        const bool last = st == order - 1;
        p.tnext = last ? nullptr : (void*)bufs[(st + 1) & 1];
        p.ld_next = w;
        p.a = (st == 0 ? 2.0 : 4.0) / lambda_max;
        p.b_cur = st == 0 ? -1.0 : -2.0;
        p.b_prev = st == 0 ? 0.0 : -1.0;
        p.y = Yc;
        p.ld_y = Rp;
        const int pending = (st + 1) - added;
        if (last || pending == 3) {
          p.cy_prev = (st >= 1 && added < st - 1) ? d[st - 1] : 0.0;
          p.cy_cur = (added < st) ? d[st] : 0.0;
          p.cy_next = d[st + 1];
          p.y_mode = added == -1 ? 1 : 2;
          added = st + 1;
        }
        p.l2pol = static_cast<unsigned>(env_int("SC_L2POL", 0));
        p.split_col = split_col;
        p.split_buf = split_col > 0 ? g->ws_split.ptr : nullptr;
        // split gather: two launches per step (first half of the columns, then the second
        // half + epilogue); the step's algorithmic bytes are counted once
        for (int part = split_col > 0 ? 1 : 0; part <= (split_col > 0 ? 2 : 0); ++part) {
          p.split_mode = part;
          p.tile_ctr = dyn_tiles_on() ? next_tile_ctr(g, s) : nullptr;
          cudaEvent_t e0 = nullptr;
          if (g_prof.on) {
            e0 = g_prof.get();
            cudaEventRecord(e0, s);
          }
          double ab = 0.0;
          SC_TRY(launch_sell_step<T>(g, p, s, g_prof.on ? &ab : nullptr));
          if (g_prof.on) {
            cudaEvent_t e1 = g_prof.get();
            cudaEventRecord(e1, s);
            g_prof.ev.emplace_back(e0, e1);
            g_prof.launches += 1;
            g_prof.step_launches += 1;
            g_prof.algo_bytes += part == 1 ? 0.0 : ab;
          }
        }
      }
      col0 += w;
      continue;
    }
    int added = -1;
    for (int st = 0; st < order; ++st) {
      StepParams p{};
      p.row_begin = 0;
      p.row_end = n;
      p.width = w;
      p.total_width = Rp;
      p.tcur = st == 0 ? (const void*)Xc : (const void*)bufs[st & 1];
      p.ld_cur = st == 0 ? Rp : w;
      p.tprev = st == 0 ? nullptr : (st == 1 ? (const void*)Xc : (const void*)bufs[(st - 1) & 1]);
      p.ld_prev = st == 1 ? Rp : w;
      const bool last = st == order - 1;
      p.tnext = last ? nullptr : (void*)bufs[(st + 1) & 1];
      p.ld_next = w;
      p.a = (st == 0 ? 2.0 : 4.0) / lambda_max;
      p.b_cur = st == 0 ? -1.0 : -2.0;
      p.b_prev = st == 0 ? 0.0 : -1.0;
      p.y = Yc;
      p.ld_y = Rp;
      const int pending = (st + 1) - added;
      if (last || pending == 3) {
        p.cy_prev = (st >= 1 && added < st - 1) ? d[st - 1] : 0.0;
        p.cy_cur = (added < st) ? d[st] : 0.0;
        p.cy_next = d[st + 1];
        p.y_mode = added == -1 ? 1 : 2;
        added = st + 1;
      }
      SC_TRY(launch_step_impl<T>(g, p, s, false, nullptr));
    }
    col0 += w;
  }
  if (!aligned) {
    copy_cols_kernel<T><<<g->num_sms * 8, 256, 0, s>>>(Yw, Rp, Y, R, n, R);
    SC_CUDA_TRY(cudaGetLastError());
    if (g_prof.on) g_prof.launches += 1;
  }
  return SC_OK;
}
template int filter_apply<float>(sc_graph*, const double*, int, double, int, const float*, float*, cudaStream_t);
template int filter_apply<double>(sc_graph*, const double*, int, double, int, const double*, double*, cudaStream_t);

// ---------------------------------------------------------------------------
// Chebyshev moments mu_0..mu_{2p} (fp64), DESIGN.md "eigencount"
// ---------------------------------------------------------------------------
// Sum of fixed-point limbs (see mom_limb in sc_sell.cu): V = sum_l acc_l 2^(32 l) mod 2^128 is
// the exact two's-complement sum of the partials x 2^80; returned as a double (V x 2^-80).
double limbs_to_double(const unsigned long long* acc) {
  unsigned __int128 v = 0;
  for (int l = 0; l < 4; ++l) v += static_cast<unsigned __int128>(acc[l]) << (32 * l);
  const bool neg = (v >> 127) != 0;
  const unsigned __int128 m = neg ? (~v + 1) : v;
  const double d = std::ldexp(static_cast<double>(static_cast<uint64_t>(m >> 64)), 64) +
                   static_cast<double>(static_cast<uint64_t>(m));
  return std::ldexp(neg ? -d : d, -80);
}

int cheb_moments(sc_graph* g, double lambda_max, int order, int R, const double* X,
                 std::vector<double>& mu, cudaStream_t s) {
  using T = double;
  constexpr int W = Vec<T>::W;
  const int64_t n = g->n_rows;
  const int Rp = (R + W - 1) / W * W;
  const T* Xw = X;
  if (Rp != R || ((uintptr_t)X % 16)) {
    SC_TRY(g->ws_sig.ensure((size_t)n * Rp * sizeof(T)));
    T* xp = g->ws_sig.as<T>();
    SC_CUDA_TRY(cudaMemsetAsync(xp, 0, (size_t)n * Rp * sizeof(T), s));
    copy_cols_kernel<T><<<g->num_sms * 8, 256, 0, s>>>(X, R, xp, Rp, n, R);
    SC_CUDA_TRY(cudaGetLastError());
    Xw = xp;
  }
  const std::vector<int> chunks = chunk_plan<T>(Rp, g->n_cols);
  int cwmax = 0;
  for (int w : chunks) cwmax = std::max(cwmax, w);
  SC_TRY(g->ws_a.ensure((size_t)g->n_cols * cwmax * sizeof(T)));
  SC_TRY(g->ws_b.ensure((size_t)g->n_cols * cwmax * sizeof(T)));
  const int max_grid = g->num_sms * 32;
  SC_TRY(g->ws_part.ensure((size_t)(max_grid * 3 + 3 * order) * sizeof(double)));
  double* part = g->ws_part.as<double>();
  double* sums = part + (size_t)max_grid * 3;   // [order][3]

  std::vector<double> acc((size_t)3 * order, 0.0);
  std::vector<double> h((size_t)3 * order);
  int col0 = 0;
  for (int w : chunks) {
    T* bufs[2] = {g->ws_b.as<T>(), g->ws_a.as<T>()};
    const T* Xc = Xw + col0;
    bool use_sell = false;
    if (sell_enabled()) SC_TRY(sell_usable<T>(g, w, 0, n, s, &use_sell));
    if (use_sell) {
      // SELL path (the filter's kernel with the moment epilogue): T_0 = the X chunk copied into
      // bufs[0] (row stride w), zero row n_cols in both buffers; the three sums of every step
      // as exact fixed-point limbs [order][3][4] (order independent: dynamic tiles stay
      // deterministic), converted on the host
      SC_TRY(g->ws_a.ensure((size_t)(g->n_cols + 1) * cwmax * sizeof(T)));
      SC_TRY(g->ws_b.ensure((size_t)(g->n_cols + 1) * cwmax * sizeof(T)));
      bufs[0] = g->ws_b.as<T>();
      bufs[1] = g->ws_a.as<T>();
      SC_TRY(g->ws_limbs.ensure(sizeof(unsigned long long) * 12 * (size_t)order));
      unsigned long long* limbs = g->ws_limbs.as<unsigned long long>();
      SC_CUDA_TRY(cudaMemsetAsync(limbs, 0, sizeof(unsigned long long) * 12 * (size_t)order, s));
      SC_CUDA_TRY(cudaMemsetAsync(bufs[0] + (size_t)g->n_cols * w, 0, sizeof(T) * w, s));
      SC_CUDA_TRY(cudaMemsetAsync(bufs[1] + (size_t)g->n_cols * w, 0, sizeof(T) * w, s));
      copy_cols_kernel<T><<<g->num_sms * 8, 256, 0, s>>>(Xc, Rp, bufs[0], w, n, w);
      SC_CUDA_TRY(cudaGetLastError());
      for (int st = 0; st < order; ++st) {
        StepParams p{};
        p.row_begin = 0;
        p.row_end = n;
        p.width = w;
        p.total_width = Rp;
        p.tcur = bufs[st & 1];
        p.ld_cur = w;
        p.tprev = st == 0 ? nullptr : (const void*)bufs[(st - 1) & 1];
        p.ld_prev = w;
        p.tnext = st == order - 1 ? nullptr : (void*)bufs[(st + 1) & 1];
        p.ld_next = w;
        p.a = (st == 0 ? 2.0 : 4.0) / lambda_max;
        p.b_cur = st == 0 ? -1.0 : -2.0;
        p.b_prev = st == 0 ? 0.0 : -1.0;
        p.mom_limbs = limbs + 12 * (size_t)st;
        p.tile_ctr = dyn_tiles_on() ? next_tile_ctr(g, s) : nullptr;
        SC_TRY(launch_sell_step<T>(g, p, s, nullptr));
      }
      std::vector<unsigned long long> hl((size_t)12 * order);
      SC_CUDA_TRY(cudaMemcpyAsync(hl.data(), limbs, sizeof(unsigned long long) * hl.size(), cudaMemcpyDeviceToHost, s));
      SC_CUDA_TRY(cudaStreamSynchronize(s));
      for (size_t i = 0; i < (size_t)3 * order; ++i) acc[i] += limbs_to_double(&hl[4 * i]);
      col0 += w;
      continue;
    }
    for (int st = 0; st < order; ++st) {
      StepParams p{};
      p.row_begin = 0;
      p.row_end = n;
      p.width = w;
      p.tcur = st == 0 ? (const void*)Xc : (const void*)bufs[st & 1];
      p.ld_cur = st == 0 ? Rp : w;
      p.tprev = st == 0 ? nullptr : (st == 1 ? (const void*)Xc : (const void*)bufs[(st - 1) & 1]);
      p.ld_prev = st == 1 ? Rp : w;
      const bool last = st == order - 1;
      p.tnext = last ? nullptr : (void*)bufs[(st + 1) & 1];
      p.ld_next = w;
      p.a = (st == 0 ? 2.0 : 4.0) / lambda_max;
      p.b_cur = st == 0 ? -1.0 : -2.0;
      p.b_prev = st == 0 ? 0.0 : -1.0;
      p.part = part;
      int grid = 0;
      SC_TRY(launch_step_impl<T>(g, p, s, true, &grid));
      if (grid > max_grid) return fail(SC_ERR_STATE, "moment partial buffer too small");
      reduce_partials_kernel<<<1, 256, 0, s>>>(part, grid, sums + 3 * st);
      SC_CUDA_TRY(cudaGetLastError());
    }
    SC_CUDA_TRY(cudaMemcpyAsync(h.data(), sums, sizeof(double) * 3 * order, cudaMemcpyDeviceToHost, s));
    SC_CUDA_TRY(cudaStreamSynchronize(s));
    for (size_t i = 0; i < h.size(); ++i) acc[i] += h[i];
    col0 += w;
  }
  // mu_0 = <T0,T0>, mu_1 = <T1,T0>; mu_{2s} = 2<Ts,Ts> - mu_0; mu_{2s+1} = 2<Ts+1,Ts> - mu_1;
  // mu_{2p} = 2<Tp,Tp> - mu_0.
  mu.assign((size_t)2 * order + 1, 0.0);
  mu[0] = acc[0];
  mu[1] = acc[1];
  for (int st = 1; st < order; ++st) {
    mu[2 * st] = 2.0 * acc[3 * st + 0] - mu[0];
    mu[2 * st + 1] = 2.0 * acc[3 * st + 1] - mu[1];
  }
  mu[2 * order] = 2.0 * acc[3 * (order - 1) + 2] - mu[0];
  return SC_OK;
}

}  // namespace sc
