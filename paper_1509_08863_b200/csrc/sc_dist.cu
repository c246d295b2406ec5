// Row-partitioned multi-GPU Chebyshev filter: the whole p-step recurrence of one rank
// in the library, halo exchange with NCCL point-to-point on a communication stream,
// overlapped with the interior rows' fused steps.
//
// BASELINE.json north_star: "the graph is row-partitioned.  Each recurrence step
// exchanges the needed rows of T_j over NVLink with NCCL ... as a halo-only exchange,
// overlapped with the interior SpMM."  The host logic that builds a rank's local CSR
// (renumbered columns: local rows first, then the halo grouped by owner; interior rows
// permuted first) and its send lists is paper_1509_08863_b200/dist.py (tested with gloo
// on CPU); this file is the per-step schedule of dist.run_filter, moved out of Python.
//
// Per step s (compute stream `cs`, communication stream `xs`):
//   pack    : send_buf <- T_s[send_idx]                      (cs)
//   exchange: ncclSend(send_buf slices) / ncclRecv(T_s halo rows, in place)   (xs, after pack)
//   interior: fused step over rows [0, n_interior)           (cs, concurrent with exchange)
//   boundary: fused step over rows [n_interior, n_local)     (cs, after the exchange)
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "sc_internal.cuh"

#define SC_NCCL_TRY(expr)                                                                   \
  do {                                                                                      \
    ncclResult_t _r = (expr);                                                               \
    if (_r != ncclSuccess) return ::sc::fail(SC_ERR_CUDA, std::string(#expr) + ": " + ncclGetErrorString(_r)); \
  } while (0)

namespace sc {
constexpr int kNcclReservedSms = 8;
}

struct sc_comm {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1, device = 0;
  cudaStream_t xs = nullptr;
  cudaEvent_t ev_pack = nullptr, ev_comm = nullptr;
};

struct sc_dist {
  sc_graph* g = nullptr;
  sc_comm* c = nullptr;
  int64_t n_local = 0, n_halo = 0, n_interior = 0, n_send = 0;
  std::vector<int64_t> send_counts, recv_counts, send_off, recv_off;
  sc::DevBuf send_idx;           // int64 [n_send] local (permuted) row positions, grouped by peer
  sc::DevBuf tA, tB, tC, sendbuf, xpad;
};

namespace sc {
namespace {

// send_buf[i][c] = T[idx[i]][c]   (w columns, row stride w)
__global__ void pack_rows_kernel(const float* __restrict__ T, const int64_t* __restrict__ idx, int64_t m, int w,
                                 float* __restrict__ out) {
  const int64_t total = m * w;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / w;
    const int c = static_cast<int>(e - i * w);
    out[e] = T[idx[i] * w + c];
  }
}

// dst[r][c] = src[r][col0 + c] for r < n, c < w (row strides lds / w)
__global__ void take_cols_kernel(const float* __restrict__ src, int64_t lds, int col0, int64_t n, int w,
                                 float* __restrict__ dst) {
  const int64_t total = n * w;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / w;
    const int c = static_cast<int>(e - r * w);
    dst[e] = src[r * lds + col0 + c];
  }
}

int exchange(sc_dist* d, float* T, int w, cudaStream_t cs) {
  sc_comm* c = d->c;
  if (c->world == 1 || (d->n_send == 0 && d->n_halo == 0)) return SC_OK;
  if (d->n_send) {
    pack_rows_kernel<<<d->g->num_sms * 4, 256, 0, cs>>>(T, d->send_idx.as<int64_t>(), d->n_send, w,
                                                         d->sendbuf.as<float>());
    SC_CUDA_TRY(cudaGetLastError());
  }
  SC_CUDA_TRY(cudaEventRecord(c->ev_pack, cs));
  SC_CUDA_TRY(cudaStreamWaitEvent(c->xs, c->ev_pack, 0));
  SC_NCCL_TRY(ncclGroupStart());
  for (int q = 0; q < c->world; ++q) {
    if (q == c->rank) continue;
    if (d->send_counts[q])
      SC_NCCL_TRY(ncclSend(d->sendbuf.as<float>() + d->send_off[q] * w, (size_t)d->send_counts[q] * w, ncclFloat, q,
                           c->comm, c->xs));
    if (d->recv_counts[q])
      SC_NCCL_TRY(ncclRecv(T + (d->n_local + d->recv_off[q]) * w, (size_t)d->recv_counts[q] * w, ncclFloat, q,
                           c->comm, c->xs));
  }
  SC_NCCL_TRY(ncclGroupEnd());
  SC_CUDA_TRY(cudaEventRecord(c->ev_comm, c->xs));
  return SC_OK;
}

}  // namespace
}  // namespace sc

using namespace sc;

extern "C" {

int sc_nccl_unique_id(void* id) {
  SC_CHECK_ARG(id, "null id");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId u;
  SC_NCCL_TRY(ncclGetUniqueId(&u));
  std::memcpy(id, &u, sizeof(u));
  return SC_OK;
}

int sc_comm_init(const void* id, int world, int rank, sc_comm** out) {
  SC_CHECK_ARG(id && out && world >= 1 && rank >= 0 && rank < world, "bad arguments");
  *out = nullptr;
  auto* c = new sc_comm();
  c->world = world;
  c->rank = rank;
  cudaGetDevice(&c->device);
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof(u));
  ncclResult_t r = ncclCommInitRank(&c->comm, world, u, rank);
  if (r != ncclSuccess) {
    delete c;
    return fail(SC_ERR_CUDA, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
  }
  if (cudaStreamCreateWithFlags(&c->xs, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_pack, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_comm, cudaEventDisableTiming) != cudaSuccess) {
    ncclCommDestroy(c->comm);
    delete c;
    return fail(SC_ERR_CUDA, "stream/event creation failed");
  }
  *out = c;
  return SC_OK;
}

int sc_comm_free(sc_comm* c) {
  if (!c) return SC_OK;
  if (c->ev_pack) cudaEventDestroy(c->ev_pack);
  if (c->ev_comm) cudaEventDestroy(c->ev_comm);
  if (c->xs) cudaStreamDestroy(c->xs);
  if (c->comm) ncclCommDestroy(c->comm);
  delete c;
  return SC_OK;
}

int sc_dist_create(sc_graph* g, sc_comm* c, int64_t n_interior, const int64_t* send_idx, int64_t n_send,
                   const int64_t* send_counts, const int64_t* recv_counts, sc_dist** out) {
  SC_CHECK_ARG(g && c && out && send_counts && recv_counts, "null argument");
  SC_CHECK_ARG(0 <= n_interior && n_interior <= g->n_rows && n_send >= 0 && (send_idx || n_send == 0), "bad sizes");
  *out = nullptr;
  auto* d = new sc_dist();
  d->g = g;
  d->c = c;
  d->n_local = g->n_rows;
  d->n_halo = g->n_cols - g->n_rows;
  d->n_interior = n_interior;
  d->n_send = n_send;
  d->send_counts.assign(send_counts, send_counts + c->world);
  d->recv_counts.assign(recv_counts, recv_counts + c->world);
  d->send_off.assign(c->world, 0);
  d->recv_off.assign(c->world, 0);
  int64_t so = 0, ro = 0;
  for (int q = 0; q < c->world; ++q) {
    d->send_off[q] = so;
    d->recv_off[q] = ro;
    so += d->send_counts[q];
    ro += d->recv_counts[q];
  }
  auto bail = [&](int rc) { delete d; return rc; };
  if (so != n_send || ro != d->n_halo) return bail(fail(SC_ERR_ARG, "send/recv counts do not match n_send / n_halo"));
  if (n_send) {
    int rc = d->send_idx.ensure(sizeof(int64_t) * n_send);
    if (rc != SC_OK) return bail(rc);
    if (cudaMemcpy(d->send_idx.ptr, send_idx, sizeof(int64_t) * n_send,
                   is_device_ptr(send_idx) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice) != cudaSuccess)
      return bail(fail(SC_ERR_CUDA, "send_idx upload failed"));
  }
  // The step kernels are persistent (grid = SMs x resident CTAs); leave a few SMs free so
  // that NCCL's send/recv kernels on the communication stream can run concurrently with
  // the interior step instead of queueing behind it.
  if (c->world > 1) g->num_sms = std::max(1, g->num_sms - kNcclReservedSms);
  *out = d;
  return SC_OK;
}

int sc_dist_free(sc_dist* d) {
  delete d;
  return SC_OK;
}

int sc_dist_filter_f32(sc_dist* d, const double* coeffs, int order, double lambda_max, int R, const float* X,
                       float* Y, void* stream) {
  SC_CHECK_ARG(d && coeffs && X && Y && order >= 1 && R >= 1 && lambda_max > 0.0, "bad arguments");
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  const int64_t nl = d->n_local, nc = d->n_local + d->n_halo;
  const size_t xbytes = sizeof(float) * nl * R;
  Staged xs_, ys_;
  SC_TRY(xs_.in(X, xbytes, cs, true));
  SC_TRY(ys_.in(Y, xbytes, cs, false));
  const float* Xd = static_cast<const float*>(xs_.dev);
  float* Yd = static_cast<float*>(ys_.dev);
  // chunk widths (multiples of 4); a ragged last group of columns goes through a padded chunk
  const int Rp = (R + 3) / 4 * 4;
  const std::vector<int> chunks = chunk_widths<float>(Rp, nc);
  int cwmax = 0;
  for (int w : chunks) cwmax = std::max(cwmax, w);
  SC_TRY(d->tA.ensure(sizeof(float) * nc * cwmax));
  SC_TRY(d->tB.ensure(sizeof(float) * nc * cwmax));
  SC_TRY(d->tC.ensure(sizeof(float) * nc * cwmax));
  SC_TRY(d->sendbuf.ensure(sizeof(float) * std::max<int64_t>(1, d->n_send) * cwmax));
  float* Yw = Yd;
  int64_t ldy = R;
  if (Rp != R) {   // Y through a padded buffer
    SC_TRY(d->xpad.ensure(sizeof(float) * nl * Rp));
    Yw = d->xpad.as<float>();
    ldy = Rp;
  }
  const int grid = d->g->num_sms * 8;
  int col0 = 0;
  for (int w : chunks) {
    float* A = d->tA.as<float>();
    float* bufs[2] = {d->tC.as<float>(), d->tB.as<float>()};   // T_j (j >= 1) in bufs[j & 1]
    // T_0 = X[:, col0 : col0 + w] (zero beyond R), halo rows filled by the step-0 exchange
    SC_CUDA_TRY(cudaMemsetAsync(A, 0, sizeof(float) * nl * w, cs));
    const int wx = std::min(w, R - col0);
    if (wx > 0) {
      if (wx == w) {
        take_cols_kernel<<<grid, 256, 0, cs>>>(Xd, R, col0, nl, w, A);
      } else {
        SC_CUDA_TRY(cudaMemcpy2DAsync(A, sizeof(float) * w, Xd + col0, sizeof(float) * R, sizeof(float) * wx, nl,
                                      cudaMemcpyDeviceToDevice, cs));
      }
      SC_CUDA_TRY(cudaGetLastError());
    }
    int added = -1;
    for (int st = 0; st < order; ++st) {
      float* cur = st == 0 ? A : bufs[st & 1];
      SC_TRY(exchange(d, cur, w, cs));
      StepParams p{};
      p.width = w;
      p.total_width = Rp;
      p.tcur = cur;
      p.ld_cur = w;
      p.tprev = st == 0 ? nullptr : (st == 1 ? (const void*)A : (const void*)bufs[(st - 1) & 1]);
      p.ld_prev = w;
      const bool last = st == order - 1;
      p.tnext = last ? nullptr : (void*)bufs[(st + 1) & 1];
      p.ld_next = w;
      p.a = (st == 0 ? 2.0 : 4.0) / lambda_max;
      p.b_cur = st == 0 ? -1.0 : -2.0;
      p.b_prev = st == 0 ? 0.0 : -1.0;
      p.y = Yw + col0;
      p.ld_y = ldy;
      const int pending = (st + 1) - added;
      if (last || pending == 3) {
        p.cy_prev = (st >= 1 && added < st - 1) ? coeffs[st - 1] : 0.0;
        p.cy_cur = (added < st) ? coeffs[st] : 0.0;
        p.cy_next = coeffs[st + 1];
        p.y_mode = added == -1 ? 1 : 2;
        added = st + 1;
      }
      p.row_begin = 0;
      p.row_end = d->n_interior;
      SC_TRY(launch_step<float>(d->g, p, cs));
      if (d->c->world > 1 && (d->n_send || d->n_halo)) SC_CUDA_TRY(cudaStreamWaitEvent(cs, d->c->ev_comm, 0));
      p.row_begin = d->n_interior;
      p.row_end = nl;
      SC_TRY(launch_step<float>(d->g, p, cs));
    }
    col0 += w;
  }
  if (Rp != R) {
    SC_CUDA_TRY(cudaMemcpy2DAsync(Yd, sizeof(float) * R, Yw, sizeof(float) * Rp, sizeof(float) * R, nl,
                                  cudaMemcpyDeviceToDevice, cs));
  }
  SC_TRY(ys_.out(Y, cs));
  return SC_OK;
}

}  // extern "C"
