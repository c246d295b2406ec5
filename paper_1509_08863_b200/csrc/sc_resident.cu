// Small-graph path of the fused Chebyshev filter: ONE cooperative launch runs all p
// recurrence steps, with each CTA's share of the CSR resident in shared memory.
//
// When the whole CSR (row offsets, column indices, weights, tile degree order) fits in
// the aggregate shared memory of the chip (148 SMs x ~200 KB), there is no reason to
// stream it from HBM p times, nor to pay a kernel launch + pipeline fill per step (for
// configs[0..2] those dominate: configs[1] gathers only ~38 MB per step).  Each CTA
// owns a contiguous range of row tiles, bulk-loads its CSR slice once, and then for
// every step runs the same fused update as cheb_step_kernel (rows of similar degree per
// warp, rolling window of 16-byte gathers, own/prev/Y rows via cp.async) followed by a
// grid-wide barrier (cooperative launch: all CTAs co-resident).
//
// PAPER.md §2.4 Eq.(3) / §4.1 step 5 (see sc_filter.cu for the recurrence).
#include <cooperative_groups.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include <cstdlib>

#include "sc_internal.cuh"

namespace cg = cooperative_groups;

namespace sc {
namespace {

constexpr unsigned FULLM = 0xffffffffu;
constexpr int kRW = 16;                 // warps per CTA
constexpr int kRThreads = kRW * 32;

template <typename T> struct RVec;
template <> struct RVec<float> {
  static constexpr int W = 4;
  // T_s is rewritten between steps inside this kernel: L2-coherent loads (ld.global.cg),
  // never the read-only / L1 path
  __device__ __forceinline__ static void ldg(const float* p, float (&v)[4]) {
    const float4 t = __ldcg(reinterpret_cast<const float4*>(p));
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  }
  __device__ __forceinline__ static void lds(const float* p, float (&v)[4]) {
    const float4 t = *reinterpret_cast<const float4*>(p);
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  }
  __device__ __forceinline__ static void st(float* p, const float (&v)[4]) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  }
};
template <> struct RVec<double> {
  static constexpr int W = 2;
  __device__ __forceinline__ static void ldg(const double* p, double (&v)[2]) {
    const double2 t = __ldcg(reinterpret_cast<const double2*>(p));
    v[0] = t.x; v[1] = t.y;
  }
  __device__ __forceinline__ static void lds(const double* p, double (&v)[2]) {
    const double2 t = *reinterpret_cast<const double2*>(p);
    v[0] = t.x; v[1] = t.y;
  }
  __device__ __forceinline__ static void st(double* p, const double (&v)[2]) {
    *reinterpret_cast<double2*>(p) = make_double2(v[0], v[1]);
  }
};

__device__ __forceinline__ void cp_async16_r(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}

struct StepCoef {   // per recurrence step
  double a, b_cur, b_prev, cy_prev, cy_cur, cy_next;
  int y_mode, pad;
};

struct ResidentParams {
  int64_t n;              // rows (= columns: single-GPU graph)
  int tr;                 // rows per tile
  int64_t ntiles;
  int order;
  const void* x;  int64_t ld_x;     // T_0 chunk
  void* buf0; void* buf1;           // T_j (j >= 1) in buf[j & 1], row stride w
  void* y;        int64_t ld_y;
  const StepCoef* coef;             // [order]
  const int64_t* tile_begin;        // [grid + 1] tile range of each CTA
  int cap_rows, cap_nnz;            // shared-memory capacity of a CTA's slice
  // stack mode (sc_stability): every T_j kept, T_j at stack + j * slot, row stride ld_stack;
  // T_0 is read from slot 0 and T_order is written (no Y)
  void* stack; int64_t slot, ld_stack;
};

template <typename T, int VPR, int EB, bool UNIT, bool STACK>
__global__ void __launch_bounds__(kRThreads, 2)
cheb_resident_kernel(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                     const float* __restrict__ val, const T* __restrict__ strength,
                     const uint16_t* __restrict__ order, ResidentParams rp) {
  constexpr int W = RVec<T>::W;
  constexpr int SW = VPR;
  constexpr int RPW = 32 / SW;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char smem[];
  // layout: rp32 [cap_rows + 1] | ord [cap_rows] | col [cap_nnz] | val [cap_nnz] | dense [kRW][3][32][16 B]
  int32_t* s_rp = reinterpret_cast<int32_t*>(smem);
  uint16_t* s_ord = reinterpret_cast<uint16_t*>(s_rp + ((rp.cap_rows + 1 + 3) & ~3));
  int32_t* s_col = reinterpret_cast<int32_t*>(s_ord + ((rp.cap_rows + 7) & ~7));
  float* s_val = reinterpret_cast<float*>(s_col + rp.cap_nnz);
  unsigned char* dense = reinterpret_cast<unsigned char*>(s_val + (UNIT ? 0 : rp.cap_nnz));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t t0 = rp.tile_begin[blockIdx.x], t1 = rp.tile_begin[blockIdx.x + 1];
  const int64_t r0 = min(t0 * rp.tr, rp.n), r1 = min(t1 * rp.tr, rp.n);
  const int64_t e0 = row_ptr[r0];
  const int nrows = static_cast<int>(r1 - r0);
  const int nnz = static_cast<int>(row_ptr[r1] - e0);
  // one-time load of this CTA's CSR slice
  for (int i = threadIdx.x; i <= nrows; i += blockDim.x) s_rp[i] = static_cast<int32_t>(row_ptr[r0 + i] - e0);
  for (int i = threadIdx.x; i < (int)((t1 - t0) * rp.tr); i += blockDim.x) s_ord[i] = order[t0 * rp.tr + i];
  for (int i = threadIdx.x; i < nnz; i += blockDim.x) {
    s_col[i] = col[e0 + i];
    if (!UNIT) s_val[i] = val[e0 + i];
  }
  __syncthreads();

  const int sub = lane / SW, sl = lane % SW, c = sl * W;
  T* d_own = reinterpret_cast<T*>(dense + ((size_t)(warp * 3 + 0) * 32 + lane) * 16);
  T* d_prv = reinterpret_cast<T*>(dense + ((size_t)(warp * 3 + 1) * 32 + lane) * 16);
  T* d_y = reinterpret_cast<T*>(dense + ((size_t)(warp * 3 + 2) * 32 + lane) * 16);
  T* y = static_cast<T*>(rp.y);
  const int nwork = static_cast<int>(t1 - t0) * kRW;   // (tile, warp) row groups of this CTA

  for (int s = 0; s < rp.order; ++s) {
    const StepCoef cf = rp.coef[s];
    const T* tcur;
    const T* tprev;
    T* tnext;
    int64_t ld_cur, ld_prev, ld_next;
    if constexpr (STACK) {
      T* st = static_cast<T*>(rp.stack);
      tcur = st + s * rp.slot;
      tprev = s == 0 ? nullptr : st + (s - 1) * rp.slot;
      tnext = st + (s + 1) * rp.slot;
      ld_cur = ld_prev = ld_next = rp.ld_stack;
    } else {
      tcur = s == 0 ? static_cast<const T*>(rp.x) : static_cast<const T*>(s & 1 ? rp.buf1 : rp.buf0);
      ld_cur = s == 0 ? rp.ld_x : (int64_t)(SW * W);
      tprev = s == 0 ? nullptr
                     : (s == 1 ? static_cast<const T*>(rp.x) : static_cast<const T*>((s - 1) & 1 ? rp.buf1 : rp.buf0));
      ld_prev = s == 1 ? rp.ld_x : (int64_t)(SW * W);
      tnext = s == rp.order - 1 ? nullptr : static_cast<T*>((s + 1) & 1 ? rp.buf1 : rp.buf0);
      ld_next = SW * W;
    }
    const char* gbase = reinterpret_cast<const char*>(tcur + c);
    const uint32_t ldb = static_cast<uint32_t>(ld_cur * sizeof(T));
    const T a = static_cast<T>(cf.a), bc = static_cast<T>(cf.b_cur), bp = static_cast<T>(cf.b_prev);
    const T cyp = static_cast<T>(cf.cy_prev), cyc = static_cast<T>(cf.cy_cur), cyn = static_cast<T>(cf.cy_next);

    for (int wk = warp; wk < nwork; wk += kRW) {
      const int tl = wk / kRW, wslot = wk - tl * kRW;
      const int rank = wslot * RPW + sub;
      const int64_t tile_r0 = (t0 + tl) * rp.tr;
      const int rows_in_tile = static_cast<int>(min((int64_t)rp.tr, rp.n - tile_r0));
      const bool valid = sub < RPW && rank < rows_in_tile;
      const int lrow = static_cast<int>(tile_r0 - r0) + (valid ? s_ord[tl * rp.tr + rank] : 0);
      const int64_t row = r0 + lrow;
      int deg = 0, b = 0;
      if (valid) {
        b = s_rp[lrow];
        deg = s_rp[lrow + 1] - b;
        cp_async16_r(d_own, tcur + row * ld_cur + c);
        if (tprev) cp_async16_r(d_prv, tprev + row * ld_prev + c);
        if (cf.y_mode == 2) cp_async16_r(d_y, y + row * rp.ld_y + c);
      }
      int maxdeg = deg;   // over the warp's rows
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) maxdeg = max(maxdeg, __shfl_xor_sync(FULLM, maxdeg, o));
      T acc[W];
#pragma unroll
      for (int w = 0; w < W; ++w) acc[w] = T(0);
      {
        const int32_t* ci = s_col + b;
        const float* wi = s_val + b;
        T g[EB][W];
        T wv[EB];
        auto issue = [&](int e, int pos) {
          const bool ok = pos < deg;
          const int k = ok ? ci[pos] : 0;
          if (!UNIT) wv[e] = ok ? static_cast<T>(wi[pos]) : T(0);
          if (ok) {
            RVec<T>::ldg(reinterpret_cast<const T*>(gbase + static_cast<uint64_t>(static_cast<uint32_t>(k)) * ldb), g[e]);
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
      }
      if (valid) {
        asm volatile("cp.async.wait_all;" ::: "memory");
        T own[W], prv[W], yv[W];
        RVec<T>::lds(d_own, own);
        if (tprev) RVec<T>::lds(d_prv, prv);
        else {
#pragma unroll
          for (int w = 0; w < W; ++w) prv[w] = T(0);
        }
        if (cf.y_mode == 2) RVec<T>::lds(d_y, yv);
        else {
#pragma unroll
          for (int w = 0; w < W; ++w) yv[w] = T(0);
        }
        const T si = strength[row];
        T tn[W];
#pragma unroll
        for (int w = 0; w < W; ++w) {
          const T lt = si * own[w] - acc[w];
          tn[w] = a * lt + bc * own[w] + bp * prv[w];
        }
        if (tnext) RVec<T>::st(tnext + row * ld_next + c, tn);
        if (cf.y_mode) {
#pragma unroll
          for (int w = 0; w < W; ++w) yv[w] += cyp * prv[w] + cyc * own[w] + cyn * tn[w];
          RVec<T>::st(y + row * rp.ld_y + c, yv);
        }
      }
    }
    if (s + 1 < rp.order) grid.sync();   // T_{s+1} complete everywhere before it is gathered
  }
}

template <typename T>
using RKernel = void (*)(const int64_t*, const int32_t*, const float*, const T*, const uint16_t*, ResidentParams);

#ifndef SC_REB_F32
#define SC_REB_F32 4   // gathers in flight per lane, resident kernel (fp32; measured best of 3-8)
#endif
template <typename T, int VPR>
RKernel<T> pick_r2(bool unit, bool stack) {
  constexpr int EB = sizeof(T) == 4 ? SC_REB_F32 : 4;
  if constexpr (sizeof(T) == 4) {   // stack mode: fp32 only (sc_stability)
    if (stack) {
      if (unit) return cheb_resident_kernel<T, VPR, EB, true, true>;
      return cheb_resident_kernel<T, VPR, EB, false, true>;
    }
  } else if (stack) {
    return nullptr;
  }
  if (unit) return cheb_resident_kernel<T, VPR, EB, true, false>;
  return cheb_resident_kernel<T, VPR, EB, false, false>;
}
template <typename T>
RKernel<T> pick_r(int vpr, bool unit, bool stack) {
  switch (vpr) {
    case 1: return pick_r2<T, 1>(unit, stack);
    case 2: return pick_r2<T, 2>(unit, stack);
    case 3: return pick_r2<T, 3>(unit, stack);
    case 4: return pick_r2<T, 4>(unit, stack);
    case 6: return pick_r2<T, 6>(unit, stack);
    case 8: return pick_r2<T, 8>(unit, stack);
    case 12: return pick_r2<T, 12>(unit, stack);
    case 16: return pick_r2<T, 16>(unit, stack);
    case 24: return pick_r2<T, 24>(unit, stack);
    case 32: return pick_r2<T, 32>(unit, stack);
    default: return nullptr;
  }
}

constexpr size_t kRSmemMax = 200 * 1024;

size_t resident_smem(int cap_rows, int cap_nnz, bool unit) {
  size_t b = sizeof(int32_t) * ((cap_rows + 1 + 3) & ~3) + sizeof(uint16_t) * ((cap_rows + 7) & ~7) +
             sizeof(int32_t) * cap_nnz + (unit ? 0 : sizeof(float) * cap_nnz);
  b = (b + 15) & ~(size_t)15;
  return b + (size_t)kRW * 3 * 32 * 16;
}

}  // namespace

static int env_int_r(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}

// Plan of the resident path for chunk width w: CTA tile ranges with their largest CSR slice.
// Returns SC_OK with *ok = false when the graph does not fit (caller uses the streaming path).
template <typename T>
int resident_filter(sc_graph* g, const double* d, int order, double lambda_max, int w, const T* Xc, int64_t ld_x,
                    T* Yc, int64_t ld_y, T* buf0, T* buf1, cudaStream_t s, bool* ok, T* stack, int64_t slot) {
  *ok = false;
  const int total_w = (int)ld_x;
  constexpr int W = sizeof(T) == 4 ? 4 : 2;
  if (w % W || g->n_cols != g->n_rows) return SC_OK;
  const int vpr = w / W;
  if (vpr < 1 || vpr > 32) return SC_OK;
  RKernel<T> k = pick_r<T>(vpr, g->unit_weights, stack != nullptr);
  if (!k) return SC_OK;
  const int tr = kRW * (32 / vpr);
  const int64_t n = g->n_rows, ntiles = (n + tr - 1) / tr;
  const auto key = std::make_pair(w | (stack ? (1 << 16) : 0), (int)sizeof(T));   // (the smem attribute is per kernel)
  auto pit = g->resident_plans.find(key);
  if (pit == g->resident_plans.end()) {
    // plan once per (graph, width): one CTA per SM (cooperative), tiles split evenly, the
    // largest CSR slice sizes the shared memory
    std::vector<int64_t> plan = {0, 0, 0, 0, 0};
    int coop = 0;
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, g->device);
    (void)0;
    // a graph whose CSR cannot fit the aggregate shared memory at one CTA per SM is never
    // resident: decide that before touching row_ptr (no device->host copy for c3 / c4)
    const size_t need = (size_t)g->nnz * (g->unit_weights ? 4 : 8) + (size_t)n * 6;
    std::vector<int64_t> rph;   // row_ptr on the host, copied once per plan
    if (coop && need <= (size_t)g->num_sms * kRSmemMax) {
      rph.resize(n + 1);
      SC_CUDA_TRY(cudaMemcpyAsync(rph.data(), g->row_ptr.as<int64_t>(), sizeof(int64_t) * (n + 1),
                                  cudaMemcpyDeviceToHost, s));
      SC_CUDA_TRY(cudaStreamSynchronize(s));
    }
    // two CTAs per SM when their slices fit (more warps to hide gather latency), else one
    for (int per_sm = 2; per_sm >= 1 && !plan[0] && !rph.empty(); --per_sm) {
      const int grid = (int)std::min<int64_t>((int64_t)g->num_sms * per_sm, ntiles);
      if (!coop || grid <= 0) break;
      std::vector<int64_t> tb(grid + 1), rpb(grid + 1);
      for (int b = 0; b <= grid; ++b) tb[b] = ntiles * b / grid;
      // balance the CTAs' step work (every step waits for the slowest CTA): boundaries where the
      // cumulative nnz + 2 x rows crosses b / grid of the total (SC_RESIDENT_BALANCE=0: equal
      // tile counts)
      if (env_int_r("SC_RESIDENT_BALANCE", 1)) {
        auto cost = [&](int64_t t) {   // cost of tiles [0, t)
          const int64_t r = std::min(t * tr, n);
          return (double)rph[r] + 2.0 * (double)r;
        };
        const double total = cost(ntiles);
        int64_t t = 0;
        for (int b = 1; b < grid; ++b) {
          const double target = total * b / grid;
          while (t < ntiles && cost(t) < target) ++t;
          tb[b] = std::max<int64_t>(tb[b - 1] + 1, std::min<int64_t>(t, ntiles - (grid - b)));
        }
        tb[grid] = ntiles;
      }
      for (int b = 0; b <= grid; ++b) rpb[b] = rph[std::min(tb[b] * tr, n)];
      int64_t cap_rows = 0, cap_nnz = 0;
      for (int b = 0; b < grid; ++b) {
        cap_rows = std::max<int64_t>(cap_rows, (tb[b + 1] - tb[b]) * tr);
        cap_nnz = std::max<int64_t>(cap_nnz, rpb[b + 1] - rpb[b]);
      }
      cap_nnz = (cap_nnz + 3) & ~int64_t(3);
      const size_t smem = resident_smem((int)cap_rows, (int)cap_nnz, g->unit_weights);
      int occ = 0;
      if (smem <= kRSmemMax &&
          cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) == cudaSuccess &&
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kRThreads, smem) == cudaSuccess &&
          occ >= per_sm) {
        auto buf = std::make_unique<DevBuf>();
        SC_TRY(buf->ensure(sizeof(int64_t) * (grid + 1)));
        SC_CUDA_TRY(cudaMemcpy(buf->ptr, tb.data(), sizeof(int64_t) * (grid + 1), cudaMemcpyHostToDevice));
        g->resident_tiles[key] = std::move(buf);
        plan = {1, grid, cap_rows, cap_nnz, (int64_t)smem};
      }
      cudaGetLastError();
    }
    pit = g->resident_plans.emplace(key, plan).first;
  }
  const std::vector<int64_t>& plan = pit->second;
  if (!plan[0]) return SC_OK;
  const int grid = (int)plan[1];
  const int cap_rows = (int)plan[2], cap_nnz = (int)plan[3];
  const size_t smem = (size_t)plan[4];
  const uint16_t* ord = tile_order(g, tr, 0, n, s);
  if (!ord) return SC_OK;
  // per-step coefficients (same schedule as filter_apply)
  std::vector<StepCoef> cf(order);
  int added = -1;
  for (int st = 0; st < order; ++st) {
    StepCoef& c = cf[st];
    std::memset(&c, 0, sizeof(c));
    c.a = (st == 0 ? 2.0 : 4.0) / lambda_max;
    c.b_cur = st == 0 ? -1.0 : -2.0;
    c.b_prev = st == 0 ? 0.0 : -1.0;
    const bool last = st == order - 1;
    if (!stack && (last || (st + 1) - added == 3)) {
      c.cy_prev = (st >= 1 && added < st - 1) ? d[st - 1] : 0.0;
      c.cy_cur = (added < st) ? d[st] : 0.0;
      c.cy_next = d[st + 1];
      c.y_mode = added == -1 ? 1 : 2;
      added = st + 1;
    }
  }
  SC_TRY(g->resident_coef.ensure(sizeof(StepCoef) * order));
  SC_CUDA_TRY(cudaMemcpyAsync(g->resident_coef.ptr, cf.data(), sizeof(StepCoef) * order, cudaMemcpyHostToDevice, s));
  ResidentParams rp{};
  rp.n = n;
  rp.tr = tr;
  rp.ntiles = ntiles;
  rp.order = order;
  rp.x = Xc;
  rp.ld_x = ld_x;
  rp.buf0 = buf0;
  rp.buf1 = buf1;
  rp.y = Yc;
  rp.ld_y = ld_y;
  rp.coef = g->resident_coef.as<StepCoef>();
  rp.tile_begin = g->resident_tiles[key]->as<int64_t>();
  rp.cap_rows = cap_rows;
  rp.cap_nnz = cap_nnz;
  rp.stack = stack;
  rp.slot = slot;
  rp.ld_stack = ld_x;
  const int64_t* a_rp = g->row_ptr.as<int64_t>();
  const int32_t* a_col = g->col_idx.as<int32_t>();
  const float* a_val = g->unit_weights ? nullptr : g->values.as<float>();
  const T* a_str = sizeof(T) == 4 ? reinterpret_cast<const T*>(g->strength32.ptr) : reinterpret_cast<const T*>(g->strength64.ptr);
  void* args[] = {(void*)&a_rp, (void*)&a_col, (void*)&a_val, (void*)&a_str, (void*)&ord, (void*)&rp};
  cudaEvent_t e0 = nullptr;
  prof_launch_begin(s, &e0);
  // (the attribute is per kernel and plans of other graphs may have set a smaller one)
  SC_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  SC_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)k, grid, kRThreads, args, smem, s));
  SC_CUDA_TRY(cudaGetLastError());
  // algorithmic bytes as for the streaming path (§0(d)): per step the CSR share of this chunk
  // (prorated by w / total_w) and the dense operands touched once
  const double csr = (double)n * 8.0 + (double)g->nnz * (g->unit_weights ? 4.0 : 8.0);
  const double dense = (double)n * w * sizeof(T) * (stack ? 3.0 : 3.0 + 2.0 / 3.0);
  prof_launch_end(s, e0, order * (csr * w / std::max(total_w, w) + dense), order);
  *ok = true;
  return SC_OK;
}
template int resident_filter<float>(sc_graph*, const double*, int, double, int, const float*, int64_t, float*, int64_t,
                                    float*, float*, cudaStream_t, bool*, float*, int64_t);
template int resident_filter<double>(sc_graph*, const double*, int, double, int, const double*, int64_t, double*,
                                     int64_t, double*, double*, cudaStream_t, bool*, double*, int64_t);

}  // namespace sc
