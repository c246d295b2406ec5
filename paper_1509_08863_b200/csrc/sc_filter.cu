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
#include <cstdlib>
#include <cstring>

#include "sc_internal.cuh"

namespace sc {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kBlock = 256;

template <typename T> struct Vec;
template <> struct Vec<float> {
  static constexpr int W = 4;
  __device__ __forceinline__ static void ldg(const float* p, float (&v)[4]) {
    float4 t = __ldg(reinterpret_cast<const float4*>(p));
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  }
  __device__ __forceinline__ static void ld(const float* p, float (&v)[4]) {
    float4 t = *reinterpret_cast<const float4*>(p);
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  }
  __device__ __forceinline__ static void st(float* p, const float (&v)[4]) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  }
};
template <> struct Vec<double> {
  static constexpr int W = 2;
  __device__ __forceinline__ static void ldg(const double* p, double (&v)[2]) {
    double2 t = __ldg(reinterpret_cast<const double2*>(p));
    v[0] = t.x; v[1] = t.y;
  }
  __device__ __forceinline__ static void ld(const double* p, double (&v)[2]) {
    double2 t = *reinterpret_cast<const double2*>(p);
    v[0] = t.x; v[1] = t.y;
  }
  __device__ __forceinline__ static void st(double* p, const double (&v)[2]) {
    *reinterpret_cast<double2*>(p) = make_double2(v[0], v[1]);
  }
};

// MOMENTS: accumulate <T_s,T_s>, <T_{s+1},T_s>, <T_{s+1},T_{s+1}> per block (fp64).
template <typename T, int VPR, int SW, int EB, bool UNIT, bool MOMENTS>
__global__ void __launch_bounds__(kBlock)
cheb_step_kernel(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                 const float* __restrict__ val, const T* __restrict__ strength, StepParams p) {
  constexpr int W = Vec<T>::W;
  constexpr int VPL = VPR / SW;   // vectors per lane
  constexpr int RPW = 32 / SW;    // rows per warp
  constexpr int EPL = EB / SW;    // column indices loaded per lane per batch
  static_assert(VPR % SW == 0 && EB % SW == 0 && 32 % SW == 0, "bad tiling");

  const int lane = threadIdx.x & 31;
  const int sub = lane / SW;
  const int sl = lane % SW;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;

  const T* tprev = static_cast<const T*>(p.tprev);   // may alias tnext (in-place rotation)
  const T* __restrict__ tcur = static_cast<const T*>(p.tcur);
  T* tnext = static_cast<T*>(p.tnext);
  T* y = static_cast<T*>(p.y);
  const T a = static_cast<T>(p.a), bc = static_cast<T>(p.b_cur), bp = static_cast<T>(p.b_prev);
  const T cyp = static_cast<T>(p.cy_prev), cyc = static_cast<T>(p.cy_cur), cyn = static_cast<T>(p.cy_next);

  double m_cc = 0.0, m_nc = 0.0, m_nn = 0.0;

  for (int64_t base = p.row_begin + warp * RPW; base < p.row_end; base += nwarps * RPW) {
    const int64_t row = base + sub;
    const bool valid = row < p.row_end;
    int64_t beg = 0;
    int deg = 0;
    if (valid) {
      beg = __ldg(row_ptr + row);
      deg = static_cast<int>(__ldg(row_ptr + row + 1) - beg);
    }

    T own[VPL][W], prv[VPL][W], acc[VPL][W];
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
      const int c = (sl + SW * v) * W;
#pragma unroll
      for (int w = 0; w < W; ++w) { own[v][w] = T(0); prv[v][w] = T(0); acc[v][w] = T(0); }
      if (valid) {
        Vec<T>::ldg(tcur + row * p.ld_cur + c, own[v]);
        if (tprev) Vec<T>::ld(tprev + row * p.ld_prev + c, prv[v]);
      }
    }

    int maxdeg = deg;
#pragma unroll
    for (int o = SW; o < 32; o <<= 1) maxdeg = max(maxdeg, __shfl_xor_sync(FULL, maxdeg, o));

    for (int off = 0; off < maxdeg; off += EB) {
      int ci[EPL];
      T wv[EPL];
#pragma unroll
      for (int t = 0; t < EPL; ++t) {
        const int pos = off + t * SW + sl;
        const bool ok = pos < deg;
        ci[t] = ok ? __ldg(col + beg + pos) : -1;
        if (UNIT) wv[t] = T(1);
        else wv[t] = ok ? static_cast<T>(__ldg(val + beg + pos)) : T(0);
      }
      T g[EB][VPL][W];
      int kk[EB];
#pragma unroll
      for (int e = 0; e < EB; ++e) {
        kk[e] = __shfl_sync(FULL, ci[e / SW], sub * SW + (e % SW));
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
          if (kk[e] >= 0) {
            Vec<T>::ldg(tcur + static_cast<int64_t>(kk[e]) * p.ld_cur + (sl + SW * v) * W, g[e][v]);
          } else {
#pragma unroll
            for (int w = 0; w < W; ++w) g[e][v][w] = T(0);
          }
        }
      }
#pragma unroll
      for (int e = 0; e < EB; ++e) {
        if (UNIT) {
#pragma unroll
          for (int v = 0; v < VPL; ++v)
#pragma unroll
            for (int w = 0; w < W; ++w) acc[v][w] += g[e][v][w];
        } else {
          const T we = __shfl_sync(FULL, wv[e / SW], sub * SW + (e % SW));
#pragma unroll
          for (int v = 0; v < VPL; ++v)
#pragma unroll
            for (int w = 0; w < W; ++w) acc[v][w] = fma(we, g[e][v][w], acc[v][w]);
        }
      }
    }

    if (valid) {
      const T si = strength[row];
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        const int c = (sl + SW * v) * W;
        T tn[W];
#pragma unroll
        for (int w = 0; w < W; ++w) {
          const T lt = si * own[v][w] - acc[v][w];            // (L T_s)[i]
          tn[w] = a * lt + bc * own[v][w] + bp * prv[v][w];   // T_{s+1}[i]
        }
        if (tnext) Vec<T>::st(tnext + row * p.ld_next + c, tn);
        if (p.y_mode) {
          T yv[W];
          if (p.y_mode == 2) Vec<T>::ld(y + row * p.ld_y + c, yv);
          else {
#pragma unroll
            for (int w = 0; w < W; ++w) yv[w] = T(0);
          }
#pragma unroll
          for (int w = 0; w < W; ++w) yv[w] += cyp * prv[v][w] + cyc * own[v][w] + cyn * tn[w];
          Vec<T>::st(y + row * p.ld_y + c, yv);
        }
        if (MOMENTS) {
#pragma unroll
          for (int w = 0; w < W; ++w) {
            const double o = own[v][w], n = tn[w];
            m_cc += o * o;
            m_nc += n * o;
            m_nn += n * n;
          }
        }
      }
    }
  }

  if (MOMENTS) {
    // deterministic block reduction: warp shuffle tree, then fixed-order warp sum
    __shared__ double red[kBlock / 32][3];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      m_cc += __shfl_xor_sync(FULL, m_cc, o);
      m_nc += __shfl_xor_sync(FULL, m_nc, o);
      m_nn += __shfl_xor_sync(FULL, m_nn, o);
    }
    if (lane == 0) {
      red[threadIdx.x >> 5][0] = m_cc;
      red[threadIdx.x >> 5][1] = m_nc;
      red[threadIdx.x >> 5][2] = m_nn;
    }
    __syncthreads();
    if (threadIdx.x < 3) {
      double s = 0.0;
      for (int w = 0; w < kBlock / 32; ++w) s += red[w][threadIdx.x];
      p.part[blockIdx.x * 3 + threadIdx.x] = s;
    }
  }
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
// tuning knobs (env SC_CHUNK, SC_EB, SC_L2_BUDGET_MB) -- see DESIGN.md
// ---------------------------------------------------------------------------
int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}

template <typename T>
using KernelFn = void (*)(const int64_t*, const int32_t*, const float*, const T*, StepParams);

template <typename T, int VPR, int EB, bool MOM>
KernelFn<T> pick_unit(bool unit) {
  constexpr int SW = VPR;                   // one 16-byte vector per lane
  constexpr int EBX = EB < SW ? SW : EB;    // at least one index per lane per batch
  if (unit) return cheb_step_kernel<T, VPR, SW, EBX, true, MOM>;
  return cheb_step_kernel<T, VPR, SW, EBX, false, MOM>;
}

template <typename T, int EB, bool MOM>
KernelFn<T> pick_vpr(int vpr, bool unit) {
  switch (vpr) {
    case 1: return pick_unit<T, 1, EB, MOM>(unit);
    case 2: return pick_unit<T, 2, EB, MOM>(unit);
    case 4: return pick_unit<T, 4, EB, MOM>(unit);
    case 8: return pick_unit<T, 8, EB, MOM>(unit);
    case 16: return pick_unit<T, 16, EB, MOM>(unit);
    case 32: return pick_unit<T, 32, EB, MOM>(unit);
    default: return nullptr;
  }
}

template <typename T>
KernelFn<T> pick_kernel(int width, bool unit, bool moments, int eb) {
  constexpr int W = Vec<T>::W;
  if (width % W) return nullptr;
  const int vpr = width / W;
  if (moments) {
    if (eb <= 8) return pick_vpr<T, 8, true>(vpr, unit);
    return pick_vpr<T, 16, true>(vpr, unit);
  }
  if (eb <= 8) return pick_vpr<T, 8, false>(vpr, unit);
  if (eb <= 16) return pick_vpr<T, 16, false>(vpr, unit);
  return pick_vpr<T, 32, false>(vpr, unit);
}

template <typename T> const T* strength_of(const sc_graph* g);
template <> const float* strength_of<float>(const sc_graph* g) { return g->strength32.as<float>(); }
template <> const double* strength_of<double>(const sc_graph* g) { return g->strength64.as<double>(); }

template <typename T>
int grid_for(KernelFn<T> k, const sc_graph* g, int64_t rows, int width) {
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kBlock, 0) != cudaSuccess || occ < 1) occ = 1;
  const int rpw = 32 / (width / Vec<T>::W);
  const int64_t need = (rows + (int64_t)(kBlock / 32) * rpw - 1) / ((int64_t)(kBlock / 32) * rpw);
  const int64_t cap = (int64_t)g->num_sms * occ;
  return static_cast<int>(std::max<int64_t>(1, std::min(need, cap)));
}

template <typename T>
int launch_step_impl(const sc_graph* g, const StepParams& p, cudaStream_t s, bool moments,
                     int* grid_out) {
  const int eb = env_int("SC_EB", 16);
  KernelFn<T> k = pick_kernel<T>(p.width, g->unit_weights, moments, eb);
  if (!k) return fail(SC_ERR_ARG, "unsupported chunk width " + std::to_string(p.width));
  const int grid = grid_for<T>(k, g, p.row_end - p.row_begin, p.width);
  if (grid_out) *grid_out = grid;
  if (p.row_end <= p.row_begin) return SC_OK;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (g_prof.on) {
    e0 = g_prof.get();
    e1 = g_prof.get();
    cudaEventRecord(e0, s);
  }
  k<<<grid, kBlock, 0, s>>>(g->row_ptr.as<int64_t>(), g->col_idx.as<int32_t>(),
                            g->unit_weights ? nullptr : g->values.as<float>(), strength_of<T>(g), p);
  SC_CUDA_TRY(cudaGetLastError());
  if (g_prof.on) {
    cudaEventRecord(e1, s);
    g_prof.ev.emplace_back(e0, e1);
    g_prof.launches += 1;
    g_prof.step_launches += 1;
    // algorithmic bytes: CSR share of this chunk + dense operands touched once
    const int64_t rows = p.row_end - p.row_begin;
    const double csr = (double)rows * 8.0 + (double)g->nnz * (g->unit_weights ? 4.0 : 8.0) * rows / g->n_rows;
    const double dense_rows = (1.0 + (p.tprev ? 1.0 : 0.0) + (p.tnext ? 1.0 : 0.0) +
                               (p.y_mode == 2 ? 2.0 : (p.y_mode == 1 ? 1.0 : 0.0)));
    const double frac = (double)p.width / (p.total_width > 0 ? p.total_width : p.width);
    g_prof.algo_bytes += csr * frac + dense_rows * (double)rows * p.width * sizeof(T);
  }
  return SC_OK;
}

// Split R columns into chunks of supported widths, each <= cw.
template <typename T>
std::vector<int> chunk_plan(int R, int64_t n_cols) {
  constexpr int W = Vec<T>::W;
  const int maxw = 32 * W;   // one warp per row
  int cw = env_int("SC_CHUNK", 0);
  if (cw <= 0) {
    // keep the gathered block T_s (plus the block being written) resident in L2
    const double budget = env_int("SC_L2_BUDGET_MB", 48) * 1048576.0;
    cw = maxw;
    while (cw > 4 * W && (double)n_cols * cw * sizeof(T) > budget) cw >>= 1;
  }
  cw = std::max(W, std::min(cw, maxw));
  std::vector<int> out;
  int rem = R;
  while (rem > 0) {
    int w = maxw;
    while (w > W && (w > rem || w > cw)) w >>= 1;
    if (w > rem) w = rem;   // only when rem < W (caller pads, so never)
    out.push_back(w);
    rem -= w;
  }
  return out;
}

}  // namespace

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

// ---------------------------------------------------------------------------
// whole filter on device buffers
// ---------------------------------------------------------------------------
template <typename T>
int filter_apply(sc_graph* g, const double* d, int order, double lambda_max, int R, const T* X,
                 T* Y, cudaStream_t s) {
  constexpr int W = Vec<T>::W;
  const int64_t n = g->n_rows;
  // operate on a vector-aligned layout; pad odd widths / misaligned pointers
  const int Rp = (R + W - 1) / W * W;
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
  const std::vector<int> chunks = chunk_plan<T>(Rp, g->n_cols);
  int cwmax = 0;
  for (int w : chunks) cwmax = std::max(cwmax, w);
  SC_TRY(g->ws_a.ensure((size_t)g->n_cols * cwmax * sizeof(T)));
  SC_TRY(g->ws_b.ensure((size_t)g->n_cols * cwmax * sizeof(T)));

  int col0 = 0;
  for (int w : chunks) {
    T* bufs[2] = {g->ws_b.as<T>(), g->ws_a.as<T>()};   // T_j lives in bufs[j & 1]
    const T* Xc = Xw + col0;
    T* Yc = Yw + col0;
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
