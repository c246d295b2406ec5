// Row-partitioned multi-GPU Chebyshev filter with the halo exchange fused into the step
// kernel: peer-to-peer stores over NVLink instead of pack + NCCL send/recv.
//
// BASELINE.json north_star: "the graph is row-partitioned.  Each recurrence step exchanges
// the needed rows of T_j over NVLink ... as a halo-only exchange, overlapped with the
// interior SpMM."  Here the exchange *is* part of the SpMM: when the fused step kernel
// (cheb_step_kernel, sc_filter.cu) finishes row i of T_{s+1}, it also stores it into the
// halo of every peer that reads row i (StepParams::p2p, P2PDev in sc_internal.cuh), so the
// transfer overlaps the arithmetic row by row and no separate exchange phase exists.
//
// Buffers.  Each rank owns three T buffers of (n_local + n_halo) x Rp floats (T_0 = A and
// the rotating T_j, j >= 1, in B / C as in sc_dist.cu), allocated with cudaMalloc so they can
// be exported with CUDA IPC; a column chunk of width w uses them with row stride w, its halo
// rows at [n_local, n_local + n_halo).  Every rank uses the same chunk plan (from n_global).
//
// Ordering (per rank, one stream; seq = a call-spanning step counter, equal on all ranks):
//   chunk start : wait(flags >= seq) [peers done with the previous chunk], T_0 = X chunk,
//                 push T_0 boundary rows into the peers' A halo, signal ++seq
//   step s      : wait(flags >= seq) [peers finished step s-1 / the push: T_s halo complete,
//                 and they no longer read the buffer this step writes into], launch the
//                 fused step (writes T_{s+1} locally and into the peers' halo), the last
//                 CTA signals ++seq
// The buffer a step writes into (T_{s+1}, which overwrites T_{s-1}) is read by a peer only in
// its steps s-1 and s+1 (halo gathers); its own step s reads T_s and its own T_{s-1} rows, so
// waiting for the peers' step s-1 before step s makes every remote store race-free.
//
// wait() is a one-warp kernel that spins (with a ~20 s watchdog that traps instead of
// hanging) on the flags the peers write with st.release.sys.  It is used only by
// sc_p2p_filter_f32, with one process per GPU.  sc_p2p_filter_group_f32 runs all ranks of a
// partition inside one process on one stream, in an order that needs no waiting (step s of
// every rank, then step s+1 ...), with the peers' buffers being ordinary device memory: the
// single-GPU emulation the tests use (no kernel ever waits on another one).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "sc_internal.cuh"

struct sc_p2p {
  sc_graph* g = nullptr;
  int rank = 0, world = 1;
  int64_t n_local = 0, n_halo = 0, n_global = 0, n_desc = 0;
  int rp_max = 0;                 // T buffers hold rp_max columns per row
  int64_t seq = 0;                // signal counter (identical on all ranks)
  sc::DevBuf buf[3];              // cudaMalloc'd (IPC-exportable)
  sc::DevBuf flags;               // int64 [world], written by the peers
  sc::DevBuf sd_ptr, sd_row, sd_peer, sd_slot, peer_nl, ctr, dev;   // dev: P2PDev
  sc::DevBuf ypad;
  sc::P2PDev host{};
  bool opened[sc::kP2PMaxWorld] = {};   // peer buffers opened with cudaIpcOpenMemHandle
  bool dirty = true;
};

namespace sc {
namespace {

// T_0 halo: for every descriptor e (row sd_row[e] -> peer sd_peer[e], slot sd_slot[e]) copy
// the w-wide row of A into the peer's A buffer; then the last CTA signals.
__global__ void p2p_push_kernel(const P2PDev* __restrict__ x, const int64_t* __restrict__ sd_row, int64_t n_desc,
                                const float* __restrict__ A, int w, int64_t signal) {
  const int w4 = w / 4;
  const int64_t total = n_desc * w4;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = t / w4;
    const int c = static_cast<int>(t - e * w4) * 4;
    const int q = x->sd_peer[e];
    const float4 v = *reinterpret_cast<const float4*>(A + sd_row[e] * w + c);
    float* dst = static_cast<float*>(x->peer_buf[0][q]) + (x->peer_nl[q] + x->sd_slot[e]) * w + c;
    *reinterpret_cast<float4*>(dst) = v;
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0 && atomicAdd(x->done_ctr, 1u) == gridDim.x - 1) {
    *x->done_ctr = 0u;
    __threadfence_system();
    for (int q = 0; q < x->world; ++q)
      if (q != x->rank)
        asm volatile("st.release.sys.global.b64 [%0], %1;" ::"l"(x->peer_flags[q] + x->rank), "l"(signal) : "memory");
  }
}

// wait until every peer published a signal >= target (multi-GPU path only)
__global__ void p2p_wait_kernel(const int64_t* __restrict__ flags, int world, int rank, int64_t target) {
  const int q = threadIdx.x;
  if (q >= world || q == rank) return;
  long long spins = 0;
  for (;;) {
    int64_t v;
    asm volatile("ld.acquire.sys.global.b64 %0, [%1];" : "=l"(v) : "l"(flags + q) : "memory");
    if (v >= target) break;
    __nanosleep(256);
    if (++spins > (40ll << 20)) __trap();   // ~20 s without progress: fail loudly, do not hang
  }
}

// dst[r][c] = src[r][col0 + c] for r < n, c < w (row strides lds / w); zero beyond wx columns
__global__ void p2p_take_cols_kernel(const float* __restrict__ src, int64_t lds, int col0, int wx, int64_t n, int w,
                                     float* __restrict__ dst) {
  const int64_t total = n * w;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / w;
    const int c = static_cast<int>(e - r * w);
    dst[e] = c < wx ? src[r * lds + col0 + c] : 0.f;
  }
}

int sync_dev(sc_p2p* p, cudaStream_t s) {
  if (!p->dirty) return SC_OK;
  SC_CUDA_TRY(cudaMemcpyAsync(p->dev.ptr, &p->host, sizeof(P2PDev), cudaMemcpyHostToDevice, s));
  SC_CUDA_TRY(cudaStreamSynchronize(s));
  p->dirty = false;
  return SC_OK;
}

// one rank's part of the per-chunk / per-step schedule
struct RankRun {
  sc_p2p* p;
  const float* X;
  float* Yw;
  int64_t ldy;
};

int chunk_start(RankRun& r, int col0, int w, int R, cudaStream_t s) {
  sc_p2p* p = r.p;
  float* A = p->buf[0].as<float>();
  const int wx = std::max(0, std::min(w, R - col0));
  p2p_take_cols_kernel<<<p->g->num_sms * 4, 256, 0, s>>>(r.X, R, col0, wx, p->n_local, w, A);
  SC_CUDA_TRY(cudaGetLastError());
  // row n_cols of every buffer (stride w): the zero row the SELL kernel's padding gathers (peers
  // store only into rows [n_local, n_cols); an earlier chunk of another width may have left
  // data here)
  const int64_t nc = p->n_local + p->n_halo;
  for (int b = 0; b < 3; ++b) SC_CUDA_TRY(cudaMemsetAsync(p->buf[b].as<float>() + nc * w, 0, sizeof(float) * w, s));
  return SC_OK;
}

int push(RankRun& r, int w, cudaStream_t s) {
  sc_p2p* p = r.p;
  const int64_t sig = ++p->seq;
  const int64_t total = std::max<int64_t>(1, p->n_desc * (w / 4));
  const int grid = (int)std::min<int64_t>((total + 255) / 256, (int64_t)p->g->num_sms * 4);
  p2p_push_kernel<<<std::max(grid, 1), 256, 0, s>>>(p->dev.as<P2PDev>(), p->sd_row.as<int64_t>(), p->n_desc,
                                                    p->buf[0].as<float>(), w, sig);
  SC_CUDA_TRY(cudaGetLastError());
  return SC_OK;
}

int wait_peers(sc_p2p* p, cudaStream_t s) {
  if (p->world == 1) return SC_OK;
  p2p_wait_kernel<<<1, 32, 0, s>>>(p->flags.as<int64_t>(), p->world, p->rank, p->seq);
  SC_CUDA_TRY(cudaGetLastError());
  return SC_OK;
}

int step(RankRun& r, const double* coeffs, int order, double lambda_max, int Rp, int col0, int w, int st, int& added,
         cudaStream_t s) {
  sc_p2p* p = r.p;
  float* A = p->buf[0].as<float>();
  float* bufs[2] = {p->buf[2].as<float>(), p->buf[1].as<float>()};   // T_j (j >= 1) in bufs[j & 1]
  const int bidx[2] = {2, 1};
  StepParams q{};
  q.width = w;
  q.total_width = Rp;
  q.tcur = st == 0 ? A : bufs[st & 1];
  q.ld_cur = w;
  q.tprev = st == 0 ? nullptr : (st == 1 ? (const void*)A : (const void*)bufs[(st - 1) & 1]);
  q.ld_prev = w;
  const bool last = st == order - 1;
  q.tnext = last ? nullptr : (void*)bufs[(st + 1) & 1];
  q.ld_next = w;
  q.a = (st == 0 ? 2.0 : 4.0) / lambda_max;
  q.b_cur = st == 0 ? -1.0 : -2.0;
  q.b_prev = st == 0 ? 0.0 : -1.0;
  q.y = r.Yw + col0;
  q.ld_y = r.ldy;
  const int pending = (st + 1) - added;
  if (last || pending == 3) {
    q.cy_prev = (st >= 1 && added < st - 1) ? coeffs[st - 1] : 0.0;
    q.cy_cur = (added < st) ? coeffs[st] : 0.0;
    q.cy_next = coeffs[st + 1];
    q.y_mode = added == -1 ? 1 : 2;
    added = st + 1;
  }
  q.row_begin = 0;
  q.row_end = p->n_local;
  q.p2p = p->world > 1 ? p->dev.as<P2PDev>() : nullptr;   // one rank: nothing to send or signal
  q.p2p_next = bidx[(st + 1) & 1];
  q.p2p_signal = ++p->seq;
  return launch_step_any<float>(p->g, q, s);
}

int prepare(sc_p2p* p, int R, float* Y, float*& Yw, int64_t& ldy, cudaStream_t s) {
  const int Rp = (R + 3) / 4 * 4;
  if (Rp > p->rp_max) return fail(SC_ERR_ARG, "R exceeds the max_R the partition was created with");
  for (int q = 0; q < p->world; ++q)
    if (q != p->rank && !p->host.peer_buf[0][q]) return fail(SC_ERR_ARG, "peer buffers not attached (import/link)");
  SC_TRY(sync_dev(p, s));
  Yw = Y;
  ldy = R;
  if (Rp != R) {
    SC_TRY(p->ypad.ensure(sizeof(float) * p->n_local * Rp));
    Yw = p->ypad.as<float>();
    ldy = Rp;
  }
  return SC_OK;
}

}  // namespace
}  // namespace sc

using namespace sc;

extern "C" {

int sc_p2p_create(sc_graph* g, int world, int rank, int64_t n_global, const int64_t* sd_ptr, const int64_t* sd_row,
                  const int32_t* sd_peer, const int64_t* sd_slot, int64_t n_desc, const int64_t* peer_n_local,
                  int max_R, sc_p2p** out) {
  SC_CHECK_ARG(g && out && peer_n_local && sd_ptr, "null argument");
  SC_CHECK_ARG(world >= 1 && world <= kP2PMaxWorld && rank >= 0 && rank < world, "1 <= world <= 8, 0 <= rank < world");
  SC_CHECK_ARG(n_desc >= 0 && (n_desc == 0 || (sd_row && sd_peer && sd_slot)), "bad descriptors");
  SC_CHECK_ARG(max_R >= 1 && n_global >= g->n_rows, "bad sizes");
  *out = nullptr;
  auto* p = new sc_p2p();
  auto bail = [&](int rc) { delete p; return rc; };
  p->g = g;
  p->rank = rank;
  p->world = world;
  p->n_local = g->n_rows;
  p->n_halo = g->n_cols - g->n_rows;
  p->n_global = n_global;
  p->n_desc = n_desc;
  p->rp_max = (max_R + 3) / 4 * 4;
  const int64_t nc = g->n_cols;
  int rc;
  for (int b = 0; b < 3; ++b) {   // + one row: the SELL kernel's zero row n_cols
    if ((rc = p->buf[b].ensure(sizeof(float) * (nc + 1) * p->rp_max)) != SC_OK) return bail(rc);
    if (cudaMemset(p->buf[b].ptr, 0, sizeof(float) * (nc + 1) * p->rp_max) != cudaSuccess)
      return bail(fail(SC_ERR_CUDA, "buffer init failed"));
  }
  if ((rc = p->flags.ensure(sizeof(int64_t) * kP2PMaxWorld)) != SC_OK) return bail(rc);
  cudaMemset(p->flags.ptr, 0, sizeof(int64_t) * kP2PMaxWorld);
  if ((rc = p->ctr.ensure(sizeof(unsigned) * 4)) != SC_OK) return bail(rc);
  cudaMemset(p->ctr.ptr, 0, sizeof(unsigned) * 4);
  auto up = [&](DevBuf& b, const void* src, size_t bytes) -> int {
    SC_TRY(b.ensure(std::max<size_t>(bytes, 8)));
    if (bytes && cudaMemcpy(b.ptr, src, bytes, is_device_ptr(src) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice) !=
                     cudaSuccess)
      return fail(SC_ERR_CUDA, "descriptor upload failed");
    return SC_OK;
  };
  if ((rc = up(p->sd_ptr, sd_ptr, sizeof(int64_t) * (p->n_local + 1))) != SC_OK) return bail(rc);
  if ((rc = up(p->sd_row, sd_row, sizeof(int64_t) * n_desc)) != SC_OK) return bail(rc);
  if ((rc = up(p->sd_peer, sd_peer, sizeof(int32_t) * n_desc)) != SC_OK) return bail(rc);
  if ((rc = up(p->sd_slot, sd_slot, sizeof(int64_t) * n_desc)) != SC_OK) return bail(rc);
  if ((rc = up(p->peer_nl, peer_n_local, sizeof(int64_t) * world)) != SC_OK) return bail(rc);
  if ((rc = p->dev.ensure(sizeof(P2PDev))) != SC_OK) return bail(rc);
  P2PDev& h = p->host;
  h.sd_ptr = p->sd_ptr.as<int64_t>();
  h.sd_peer = p->sd_peer.as<int32_t>();
  h.sd_slot = p->sd_slot.as<int64_t>();
  h.peer_nl = p->peer_nl.as<int64_t>();
  h.done_ctr = p->ctr.as<unsigned>();
  h.rank = rank;
  h.world = world;
  // first row with descriptors (the boundary block of an interior-first local order)
  h.row0 = p->n_local;
  if (n_desc) {
    std::vector<int64_t> ptr(p->n_local + 1);
    if (cudaMemcpy(ptr.data(), p->sd_ptr.ptr, sizeof(int64_t) * (p->n_local + 1), cudaMemcpyDeviceToHost) != cudaSuccess)
      return bail(fail(SC_ERR_CUDA, "descriptor readback failed"));
    int64_t i = 0;
    while (i < p->n_local && ptr[i + 1] == ptr[i]) ++i;
    h.row0 = i;
  }
  for (int b = 0; b < 3; ++b) h.peer_buf[b][rank] = p->buf[b].ptr;
  h.peer_flags[rank] = p->flags.as<int64_t>();
  *out = p;
  return SC_OK;
}

int sc_p2p_free(sc_p2p* p) {
  if (!p) return SC_OK;
  for (int q = 0; q < p->world; ++q) {
    if (!p->opened[q]) continue;
    for (int b = 0; b < 3; ++b)
      if (p->host.peer_buf[b][q]) cudaIpcCloseMemHandle(p->host.peer_buf[b][q]);
    if (p->host.peer_flags[q]) cudaIpcCloseMemHandle(p->host.peer_flags[q]);
  }
  delete p;
  return SC_OK;
}

int sc_p2p_export(sc_p2p* p, void* handles) {
  SC_CHECK_ARG(p && handles, "null argument");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  auto* h = static_cast<cudaIpcMemHandle_t*>(handles);
  for (int b = 0; b < 3; ++b) SC_CUDA_TRY(cudaIpcGetMemHandle(&h[b], p->buf[b].ptr));
  SC_CUDA_TRY(cudaIpcGetMemHandle(&h[3], p->flags.ptr));
  return SC_OK;
}

int sc_p2p_import(sc_p2p* p, int peer, const void* handles) {
  SC_CHECK_ARG(p && handles && peer >= 0 && peer < p->world && peer != p->rank, "bad arguments");
  const auto* h = static_cast<const cudaIpcMemHandle_t*>(handles);
  void* ptr = nullptr;
  for (int b = 0; b < 3; ++b) {
    SC_CUDA_TRY(cudaIpcOpenMemHandle(&ptr, h[b], cudaIpcMemLazyEnablePeerAccess));
    p->host.peer_buf[b][peer] = ptr;
  }
  SC_CUDA_TRY(cudaIpcOpenMemHandle(&ptr, h[3], cudaIpcMemLazyEnablePeerAccess));
  p->host.peer_flags[peer] = static_cast<int64_t*>(ptr);
  p->opened[peer] = true;
  p->dirty = true;
  return SC_OK;
}

int sc_p2p_link_local(sc_p2p* p, sc_p2p* peer) {
  SC_CHECK_ARG(p && peer && p != peer && p->world == peer->world && peer->rank != p->rank, "bad arguments");
  for (int b = 0; b < 3; ++b) p->host.peer_buf[b][peer->rank] = peer->buf[b].ptr;
  p->host.peer_flags[peer->rank] = peer->flags.as<int64_t>();
  p->dirty = true;
  return SC_OK;
}

int sc_p2p_filter_f32(sc_p2p* p, const double* coeffs, int order, double lambda_max, int R, const float* X, float* Y,
                      void* stream) {
  SC_CHECK_ARG(p && coeffs && X && Y && order >= 1 && R >= 1 && lambda_max > 0.0, "bad arguments");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t xbytes = sizeof(float) * p->n_local * R;
  Staged xs_, ys_;
  SC_TRY(xs_.in(X, xbytes, s, true));
  SC_TRY(ys_.in(Y, xbytes, s, false));
  float* Yw;
  int64_t ldy;
  SC_TRY(prepare(p, R, static_cast<float*>(ys_.dev), Yw, ldy, s));
  RankRun r{p, static_cast<const float*>(xs_.dev), Yw, ldy};
  const int Rp = (R + 3) / 4 * 4;
  const std::vector<int> chunks = chunk_widths<float>(Rp, p->n_global);
  int col0 = 0;
  for (int w : chunks) {
    SC_TRY(wait_peers(p, s));   // peers done with the previous chunk / call
    SC_TRY(chunk_start(r, col0, w, R, s));
    SC_TRY(push(r, w, s));
    int added = -1;
    for (int st = 0; st < order; ++st) {
      SC_TRY(wait_peers(p, s));
      SC_TRY(step(r, coeffs, order, lambda_max, Rp, col0, w, st, added, s));
    }
    col0 += w;
  }
  if (Rp != R)
    SC_CUDA_TRY(cudaMemcpy2DAsync(ys_.dev, sizeof(float) * R, Yw, sizeof(float) * Rp, sizeof(float) * R, p->n_local,
                                  cudaMemcpyDeviceToDevice, s));
  SC_TRY(ys_.out(Y, s));
  return SC_OK;
}

int sc_p2p_filter_group_f32(sc_p2p* const* ps, int world, const double* coeffs, int order, double lambda_max, int R,
                            const float* const* X, float* const* Y, void* stream) {
  SC_CHECK_ARG(ps && X && Y && coeffs && world >= 1 && world <= kP2PMaxWorld && order >= 1 && R >= 1 &&
                   lambda_max > 0.0,
               "bad arguments");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  std::vector<RankRun> runs(world);
  for (int q = 0; q < world; ++q) {
    SC_CHECK_ARG(ps[q] && ps[q]->rank == q && ps[q]->world == world && X[q] && Y[q], "ranks must be 0..world-1");
    SC_CHECK_ARG(is_device_ptr(X[q]) && is_device_ptr(Y[q]), "device buffers required");
    float* Yw;
    int64_t ldy;
    SC_TRY(prepare(ps[q], R, Y[q], Yw, ldy, s));
    runs[q] = RankRun{ps[q], X[q], Yw, ldy};
  }
  const int Rp = (R + 3) / 4 * 4;
  const std::vector<int> chunks = chunk_widths<float>(Rp, ps[0]->n_global);
  // SC_P2P_GROUP_WAITS=1 (tests): also launch every rank's flag wait where the multi-process
  // path does.  In this order each wait's flags were published by kernels that precede it on
  // the stream, so it returns at once -- it checks the signal protocol without any kernel
  // waiting for another one to be scheduled.
  const bool waits = std::getenv("SC_P2P_GROUP_WAITS") && std::atoi(std::getenv("SC_P2P_GROUP_WAITS")) != 0;
  int col0 = 0;
  for (int w : chunks) {
    for (int q = 0; q < world; ++q) SC_TRY(chunk_start(runs[q], col0, w, R, s));
    for (int q = 0; q < world; ++q) {
      if (waits) SC_TRY(wait_peers(ps[q], s));
      SC_TRY(push(runs[q], w, s));
    }
    std::vector<int> added(world, -1);
    for (int st = 0; st < order; ++st)
      for (int q = 0; q < world; ++q) {
        if (waits) SC_TRY(wait_peers(ps[q], s));
        SC_TRY(step(runs[q], coeffs, order, lambda_max, Rp, col0, w, st, added[q], s));
      }
    col0 += w;
  }
  for (int q = 0; q < world; ++q) {
    sc_p2p* p = ps[q];
    if (Rp != R)
      SC_CUDA_TRY(cudaMemcpy2DAsync(Y[q], sizeof(float) * R, runs[q].Yw, sizeof(float) * Rp, sizeof(float) * R,
                                    p->n_local, cudaMemcpyDeviceToDevice, s));
  }
  SC_CUDA_TRY(cudaStreamSynchronize(s));
  return SC_OK;
}

}  // extern "C"
