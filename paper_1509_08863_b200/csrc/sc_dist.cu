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
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <thread>
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
  sc::DevBuf lz, probes, mpart, msums;   // partitioned lambda estimates (Lanczos, moments)
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
  if (!c->comm) return fail(SC_ERR_ARG, "a local (emulation) communicator has no NCCL exchange");
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


// ---------------------------------------------------------------------------
// Row-partitioned lambda estimates (§4.1 steps 1-2, l.309-311): Lanczos for
// lambda_N and the Chebyshev moments of the eigencount (§3.2 l.269-275) on the partition.
// The same SpMV / fused-step kernels as one GPU, with (a) the halo of the vector filled
// before every product and (b) every inner product summed over the ranks.  `Ranks` are the
// plans this process holds: one (one process per GPU: NCCL send/recv halos, NCCL all-reduce)
// or all of them (the single-GPU emulation the tests use: halo rows copied between the ranks'
// buffers, sums taken in rank order).
// ---------------------------------------------------------------------------
struct Ranks {
  std::vector<sc_dist*> d;
  int world() const { return d[0]->c->world; }
  bool nccl() const { return d.size() == 1 && world() > 1; }
};

struct DPtrs {
  double* p[kP2PMaxWorld];
};

// x[r][0..count) = sum over ranks in rank order, written back to every rank
__global__ void sum_ranks_kernel(DPtrs x, int world, int count) {
  for (int i = threadIdx.x; i < count; i += blockDim.x) {
    double acc = 0.0;
    for (int r = 0; r < world; ++r) acc += x.p[r][i];
    for (int r = 0; r < world; ++r) x.p[r][i] = acc;
  }
}

int allreduce_sum(const Ranks& R, const std::vector<double*>& x, int count, cudaStream_t s) {
  if (R.world() == 1) return SC_OK;
  if (R.nccl()) {
    SC_NCCL_TRY(ncclAllReduce(x[0], x[0], count, ncclDouble, ncclSum, R.d[0]->c->comm, s));
    return SC_OK;
  }
  DPtrs dp{};
  for (size_t r = 0; r < x.size(); ++r) dp.p[r] = x[r];
  sum_ranks_kernel<<<1, 256, 0, s>>>(dp, static_cast<int>(x.size()), count);
  SC_CUDA_TRY(cudaGetLastError());
  return SC_OK;
}

// halo rows of every held rank's buffer (row stride w floats; fp64 rows travel as 2 floats
// per double, bit for bit)
int halo_fill(const Ranks& R, const std::vector<float*>& T, int w, cudaStream_t s) {
  if (R.world() == 1) return SC_OK;
  if (R.nccl()) {
    sc_dist* d = R.d[0];
    SC_TRY(d->sendbuf.ensure(sizeof(float) * std::max<int64_t>(1, d->n_send) * w));
    SC_TRY(exchange(d, T[0], w, s));
    if (d->n_send || d->n_halo) SC_CUDA_TRY(cudaStreamWaitEvent(s, d->c->ev_comm, 0));
    return SC_OK;
  }
  const int world = R.world();
  for (int r = 0; r < world; ++r)
    for (int q = 0; q < world; ++q) {
      if (q == r) continue;
      sc_dist* dr = R.d[r];
      sc_dist* dq = R.d[q];
      const int64_t cnt = dr->recv_counts[q];
      if (cnt != dq->send_counts[r]) return fail(SC_ERR_ARG, "send / receive counts of two ranks disagree");
      if (!cnt) continue;
      pack_rows_kernel<<<dr->g->num_sms * 2, 256, 0, s>>>(T[q], dq->send_idx.as<int64_t>() + dq->send_off[r], cnt, w,
                                                           T[r] + (dr->n_local + dr->recv_off[q]) * w);
      SC_CUDA_TRY(cudaGetLastError());
    }
  return SC_OK;
}

int ranks_of(sc_dist* const* ds, int nheld, Ranks* R) {
  SC_CHECK_ARG(ds && nheld >= 1, "null plans");
  R->d.assign(ds, ds + nheld);
  const int world = ds[0]->c->world;
  if (nheld == 1) {
    SC_CHECK_ARG(world == 1 || ds[0]->c->comm, "one held rank of a multi-rank partition needs an NCCL communicator");
    return SC_OK;
  }
  SC_CHECK_ARG(nheld == world && world <= kP2PMaxWorld, "hold one rank or all ranks of the partition");
  for (int r = 0; r < nheld; ++r)
    SC_CHECK_ARG(ds[r] && ds[r]->c->world == world && ds[r]->c->rank == r, "plans must be ranks 0..world-1 in order");
  return SC_OK;
}

// Lanczos (fp64) on the partition: theta = largest Ritz value of L after `iters` steps.  The
// start vector of rank r's local row i is the counter generator's (seed, stream 0) entry
// row0[r] + i.
int dist_lanczos(const Ranks& R, int iters, uint64_t seed, const int64_t* row0, double* theta, cudaStream_t s) {
  const int nh = static_cast<int>(R.d.size());
  struct Buf { double *v, *vprev, *w, *tmp, *part, *alpha, *b2, *beta; };
  std::vector<Buf> b(nh);
  for (int r = 0; r < nh; ++r) {
    sc_dist* d = R.d[r];
    const size_t nc = (size_t)(d->n_local + d->n_halo), nl = (size_t)d->n_local;
    SC_TRY(d->lz.ensure(sizeof(double) * (2 * nc + 2 * nl + lz::kDotBlocks + 3 * (size_t)(iters + 2))));
    double* base = d->lz.as<double>();
    b[r].v = base;
    b[r].vprev = b[r].v + nc;
    b[r].w = b[r].vprev + nc;
    b[r].tmp = b[r].w + nl;
    b[r].part = b[r].tmp + nl;
    b[r].alpha = b[r].part + lz::kDotBlocks;
    b[r].b2 = b[r].alpha + (iters + 2);
    b[r].beta = b[r].b2 + (iters + 2);
    SC_CUDA_TRY(cudaMemsetAsync(b[r].v, 0, sizeof(double) * 2 * nc, s));
  }
  auto scal = [&](double* Buf::*field, int j) {
    std::vector<double*> x(nh);
    for (int r = 0; r < nh; ++r) x[r] = (b[r].*field) + j;
    return x;
  };
  auto vecs = [&](double* Buf::*field) {
    std::vector<float*> x(nh);
    for (int r = 0; r < nh; ++r) x[r] = reinterpret_cast<float*>(b[r].*field);
    return x;
  };
  // v_0 = r / ||r||
  for (int r = 0; r < nh; ++r) {
    sc_dist* d = R.d[r];
    SC_TRY(random_signals<double>(d->n_local, 1, row0 ? row0[r] : 0, seed, 0, 1.0, b[r].tmp, s));
    SC_TRY(lz::dot_local(b[r].tmp, b[r].tmp, d->n_local, b[r].part, b[r].b2, s));
  }
  SC_TRY(allreduce_sum(R, scal(&Buf::b2, 0), 1, s));
  for (int r = 0; r < nh; ++r) {
    SC_TRY(lz::scale_inv_sqrt(b[r].v, b[r].tmp, b[r].b2, nullptr, R.d[r]->n_local, s));
    SC_CUDA_TRY(cudaMemsetAsync(b[r].beta, 0, sizeof(double), s));
  }
  for (int j = 0; j < iters; ++j) {
    SC_TRY(halo_fill(R, vecs(&Buf::v), 2, s));
    for (int r = 0; r < nh; ++r) {
      SC_TRY(lz::spmv(R.d[r]->g, b[r].v, j ? b[r].vprev : nullptr, b[r].beta + j, b[r].w, s));
      SC_TRY(lz::dot_local(b[r].w, b[r].v, R.d[r]->n_local, b[r].part, b[r].alpha + j, s));
    }
    SC_TRY(allreduce_sum(R, scal(&Buf::alpha, j), 1, s));
    for (int r = 0; r < nh; ++r) {
      SC_TRY(lz::axpy_neg(b[r].w, b[r].v, b[r].alpha + j, R.d[r]->n_local, s));
      SC_TRY(lz::dot_local(b[r].w, b[r].w, R.d[r]->n_local, b[r].part, b[r].b2 + j + 1, s));
    }
    SC_TRY(allreduce_sum(R, scal(&Buf::b2, j + 1), 1, s));
    for (int r = 0; r < nh; ++r) {
      std::swap(b[r].vprev, b[r].v);
      SC_TRY(lz::scale_inv_sqrt(b[r].v, b[r].w, b[r].b2 + j + 1, b[r].beta + j + 1, R.d[r]->n_local, s));
    }
  }
  std::vector<double> ha(iters), hb(iters + 1);
  SC_CUDA_TRY(cudaMemcpyAsync(ha.data(), b[0].alpha, sizeof(double) * iters, cudaMemcpyDeviceToHost, s));
  SC_CUDA_TRY(cudaMemcpyAsync(hb.data(), b[0].beta, sizeof(double) * (iters + 1), cudaMemcpyDeviceToHost, s));
  SC_CUDA_TRY(cudaStreamSynchronize(s));
  *theta = lz::theta_from(ha, hb);
  return SC_OK;
}

// max over ranks of the local strengths (Gershgorin: lambda_N <= 2 max_i s_i)
int dist_max_strength(const Ranks& R, double* out, cudaStream_t s) {
  double m = 0.0;
  for (sc_dist* d : R.d) m = std::max(m, d->g->max_strength);
  if (R.nccl()) {
    sc_dist* d = R.d[0];
    SC_TRY(d->msums.ensure(sizeof(double)));
    SC_CUDA_TRY(cudaMemcpyAsync(d->msums.ptr, &m, sizeof(double), cudaMemcpyHostToDevice, s));
    SC_NCCL_TRY(ncclAllReduce(d->msums.ptr, d->msums.ptr, 1, ncclDouble, ncclMax, d->c->comm, s));
    SC_CUDA_TRY(cudaMemcpyAsync(&m, d->msums.ptr, sizeof(double), cudaMemcpyDeviceToHost, s));
    SC_CUDA_TRY(cudaStreamSynchronize(s));
  }
  *out = m;
  return SC_OK;
}

// dst[r][c] = c < cols_left ? src[r * lds + col0 + c] : 0   (fp64, w columns)
__global__ void take_cols_d_kernel(const double* __restrict__ src, int64_t lds, int col0, int cols_left, int64_t n,
                                   int w, double* __restrict__ dst) {
  const int64_t total = n * w;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / w;
    const int c = static_cast<int>(e - r * w);
    dst[e] = c < cols_left ? src[r * lds + col0 + c] : 0.0;
  }
}

// Chebyshev moments mu_0..mu_{2p} of the probes X (n_probe columns, N(0, 1/n_probe) entries
// from the counter generator, stream 2, counters (row0[r] + i) * n_probe + q) on the partition;
// the same identity as cheb_moments (sc_filter.cu) on the sums over all ranks
int dist_moments(const Ranks& R, double lambda_max, int order, int np, uint64_t seed, const int64_t* row0,
                 std::vector<double>& mu, cudaStream_t s) {
  const int nh = static_cast<int>(R.d.size());
  // fixed chunk plan, equal on every rank (the exchanges are collective): 16-double chunks
  std::vector<int> chunks;
  {
    int rem = (np + 1) / 2;   // in 16-byte vectors of 2 doubles
    const int set[] = {8, 6, 4, 3, 2, 1};
    while (rem > 0) {
      int v = 1;
      for (int c : set)
        if (c <= rem) { v = c; break; }
      chunks.push_back(2 * v);
      rem -= v;
    }
  }
  int cwmax = 0;
  for (int w : chunks) cwmax = std::max(cwmax, w);
  const int max_grid = 148 * 32;
  std::vector<double*> sums(nh);
  for (int r = 0; r < nh; ++r) {
    sc_dist* d = R.d[r];
    const int64_t nc = d->n_local + d->n_halo;
    SC_TRY(d->probes.ensure(sizeof(double) * std::max<int64_t>(1, d->n_local) * np));
    SC_TRY(d->tA.ensure(sizeof(double) * nc * cwmax));
    SC_TRY(d->tB.ensure(sizeof(double) * nc * cwmax));
    SC_TRY(d->tC.ensure(sizeof(double) * nc * cwmax));
    SC_TRY(d->mpart.ensure(sizeof(double) * 2 * max_grid * 3));
    SC_TRY(d->msums.ensure(sizeof(double) * (size_t)order * 6));
    SC_CUDA_TRY(cudaMemsetAsync(d->msums.ptr, 0, sizeof(double) * (size_t)order * 6, s));
    if (d->n_local) SC_TRY(random_signals<double>(d->n_local, np, row0 ? row0[r] : 0, seed, 2, 1.0 / np,
                                                  d->probes.as<double>(), s));
    sums[r] = d->msums.as<double>();
  }
  std::vector<double> acc((size_t)order * 3, 0.0), h((size_t)order * 6);
  int col0 = 0;
  for (int w : chunks) {
    std::vector<double*> A(nh), B(nh), C(nh);
    for (int r = 0; r < nh; ++r) {
      sc_dist* d = R.d[r];
      A[r] = d->tA.as<double>();
      B[r] = d->tB.as<double>();
      C[r] = d->tC.as<double>();
      SC_CUDA_TRY(cudaMemsetAsync(A[r], 0, sizeof(double) * (d->n_local + d->n_halo) * w, s));
      if (d->n_local) {
        take_cols_d_kernel<<<d->g->num_sms * 4, 256, 0, s>>>(d->probes.as<double>(), np, col0, np - col0, d->n_local,
                                                             w, A[r]);
        SC_CUDA_TRY(cudaGetLastError());
      }
      SC_CUDA_TRY(cudaMemsetAsync(sums[r], 0, sizeof(double) * (size_t)order * 6, s));
    }
    for (int st = 0; st < order; ++st) {
      std::vector<float*> cur(nh);
      for (int r = 0; r < nh; ++r) cur[r] = reinterpret_cast<float*>(st == 0 ? A[r] : ((st & 1) ? B[r] : C[r]));
      SC_TRY(halo_fill(R, cur, 2 * w, s));
      for (int r = 0; r < nh; ++r) {
        sc_dist* d = R.d[r];
        double* bufs[2] = {C[r], B[r]};   // T_j (j >= 1) in bufs[j & 1]
        StepParams p{};
        p.width = w;
        p.total_width = w;
        p.tcur = cur[r];
        p.ld_cur = w;
        p.tprev = st == 0 ? nullptr : (st == 1 ? (const void*)A[r] : (const void*)bufs[(st - 1) & 1]);
        p.ld_prev = w;
        p.tnext = st == order - 1 ? nullptr : (void*)bufs[(st + 1) & 1];
        p.ld_next = w;
        p.a = (st == 0 ? 2.0 : 4.0) / lambda_max;
        p.b_cur = st == 0 ? -1.0 : -2.0;
        p.b_prev = st == 0 ? 0.0 : -1.0;
        const int64_t bounds[3] = {0, d->n_interior, d->n_local};
        for (int part = 0; part < 2; ++part) {
          if (bounds[part + 1] <= bounds[part]) continue;
          p.row_begin = bounds[part];
          p.row_end = bounds[part + 1];
          p.part = d->mpart.as<double>() + (size_t)part * max_grid * 3;
          int grid = 0;
          SC_TRY(launch_moments_step(d->g, p, s, &grid));
          if (grid > max_grid) return fail(SC_ERR_STATE, "moment partial buffer too small");
          SC_TRY(reduce_moment_partials(p.part, grid, sums[r] + (size_t)st * 6 + 3 * part, s));
        }
      }
    }
    SC_TRY(allreduce_sum(R, sums, order * 6, s));
    SC_CUDA_TRY(cudaMemcpyAsync(h.data(), sums[0], sizeof(double) * h.size(), cudaMemcpyDeviceToHost, s));
    SC_CUDA_TRY(cudaStreamSynchronize(s));
    for (int st = 0; st < order; ++st)
      for (int c = 0; c < 3; ++c) acc[(size_t)st * 3 + c] += h[(size_t)st * 6 + c] + h[(size_t)st * 6 + 3 + c];
    col0 += w;
  }
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

// ---------------------------------------------------------------------------
// Collectives of the distributed k-means (Coll, sc_internal.cuh)
// ---------------------------------------------------------------------------
struct NcclColl : Coll {
  ncclComm_t comm;
  NcclColl(ncclComm_t c, int r, int w) : comm(c) { rank = r; world = w; }
  int red(void* p, size_t n, ncclDataType_t t, ncclRedOp_t op, cudaStream_t s) {
    if (world == 1 || n == 0) return SC_OK;
    SC_NCCL_TRY(ncclAllReduce(p, p, n, t, op, comm, s));
    return SC_OK;
  }
  int sum_u64(unsigned long long* p, size_t n, cudaStream_t s) override { return red(p, n, ncclUint64, ncclSum, s); }
  int sum_u32(unsigned* p, size_t n, cudaStream_t s) override { return red(p, n, ncclUint32, ncclSum, s); }
  int sum_i32(int* p, size_t n, cudaStream_t s) override { return red(p, n, ncclInt32, ncclSum, s); }
  int sum_f64(double* p, size_t n, cudaStream_t s) override { return red(p, n, ncclFloat64, ncclSum, s); }
  int max_u32(unsigned* p, size_t n, cudaStream_t s) override { return red(p, n, ncclUint32, ncclMax, s); }
};

// Single-process emulation: one host thread per rank, each on its own stream of the one GPU.
// A reduction synchronises the rank's stream, deposits its buffer in a host slot, meets the
// other ranks at a host barrier, reduces the slots in rank order and copies the result back --
// the ranks wait for each other on the host only (no kernel waits for another rank).
struct LocalGroup {
  int world;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long gen = 0;
  bool failed = false;
  std::vector<std::vector<unsigned char>> slot;
  explicit LocalGroup(int w) : world(w), slot(w) {}
  bool barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long long g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g || failed; });
    }
    return !failed;
  }
  void fail_all() {
    std::lock_guard<std::mutex> lk(mu);
    failed = true;
    cv.notify_all();
  }
};

struct LocalColl : Coll {
  LocalGroup* grp;
  LocalColl(LocalGroup* g, int r) : grp(g) { rank = r; world = g->world; }
  template <typename T, typename Op>
  int red(T* p, size_t n, cudaStream_t s, Op op) {
    if (world == 1 || n == 0) return SC_OK;
    std::vector<unsigned char>& mine = grp->slot[rank];
    mine.resize(n * sizeof(T));
    SC_CUDA_TRY(cudaMemcpyAsync(mine.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost, s));
    SC_CUDA_TRY(cudaStreamSynchronize(s));
    if (!grp->barrier()) return fail(SC_ERR_STATE, "another emulated rank failed");
    std::vector<T> out(n);
    std::memcpy(out.data(), grp->slot[0].data(), n * sizeof(T));
    for (int r = 1; r < world; ++r) {
      const T* x = reinterpret_cast<const T*>(grp->slot[r].data());
      for (size_t i = 0; i < n; ++i) out[i] = op(out[i], x[i]);
    }
    if (!grp->barrier()) return fail(SC_ERR_STATE, "another emulated rank failed");
    SC_CUDA_TRY(cudaMemcpyAsync(p, out.data(), n * sizeof(T), cudaMemcpyHostToDevice, s));
    SC_CUDA_TRY(cudaStreamSynchronize(s));
    return SC_OK;
  }
  int sum_u64(unsigned long long* p, size_t n, cudaStream_t s) override {
    return red(p, n, s, [](unsigned long long a, unsigned long long b) { return a + b; });
  }
  int sum_u32(unsigned* p, size_t n, cudaStream_t s) override {
    return red(p, n, s, [](unsigned a, unsigned b) { return a + b; });
  }
  int sum_i32(int* p, size_t n, cudaStream_t s) override { return red(p, n, s, [](int a, int b) { return a + b; }); }
  int sum_f64(double* p, size_t n, cudaStream_t s) override {
    return red(p, n, s, [](double a, double b) { return a + b; });
  }
  int max_u32(unsigned* p, size_t n, cudaStream_t s) override {
    return red(p, n, s, [](unsigned a, unsigned b) { return a > b ? a : b; });
  }
};
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

int sc_comm_local(int world, int rank, sc_comm** out) {
  SC_CHECK_ARG(out && world >= 1 && world <= kP2PMaxWorld && rank >= 0 && rank < world, "bad arguments");
  auto* c = new sc_comm();
  c->world = world;
  c->rank = rank;
  cudaGetDevice(&c->device);
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
  if (c->world > 1 && c->comm) g->num_sms = std::max(1, g->num_sms - kNcclReservedSms);
  *out = d;
  return SC_OK;
}

int sc_dist_free(sc_dist* d) {
  if (d && d->g && d->c && d->c->world > 1 && d->c->comm) d->g->num_sms += kNcclReservedSms;   // as before create
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
  // + one row: the all-zero row n_cols that the SELL kernel's padding gathers
  SC_TRY(d->tA.ensure(sizeof(float) * (nc + 1) * cwmax));
  SC_TRY(d->tB.ensure(sizeof(float) * (nc + 1) * cwmax));
  SC_TRY(d->tC.ensure(sizeof(float) * (nc + 1) * cwmax));
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
    for (float* b : {A, bufs[0], bufs[1]}) SC_CUDA_TRY(cudaMemsetAsync(b + nc * w, 0, sizeof(float) * w, cs));
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
      SC_TRY(launch_step_any<float>(d->g, p, cs));
      if (d->c->world > 1 && (d->n_send || d->n_halo)) SC_CUDA_TRY(cudaStreamWaitEvent(cs, d->c->ev_comm, 0));
      p.row_begin = d->n_interior;
      p.row_end = nl;
      SC_TRY(launch_step_any<float>(d->g, p, cs));
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

int sc_dist_lambda_max(sc_dist* const* ds, int nheld, int iters, double margin, uint64_t seed, const int64_t* row0,
                       double* out, void* stream) {
  SC_CHECK_ARG(out && iters >= 1 && margin >= 0.0, "bad arguments");
  Ranks R;
  SC_TRY(ranks_of(ds, nheld, &R));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double theta = 0.0, smax = 0.0;
  SC_TRY(dist_lanczos(R, iters, seed, row0, &theta, s));
  SC_TRY(dist_max_strength(R, &smax, s));
  const double gersh = 2.0 * smax;
  double b = (1.0 + margin) * theta;
  if (!(b > 0.0) || b > gersh) b = gersh;
  if (!(b > 0.0)) b = 1.0;
  *out = b;
  return SC_OK;
}

int sc_dist_cheb_moments(sc_dist* const* ds, int nheld, double lambda_max, int order, int n_probe, uint64_t seed,
                         const int64_t* row0, double* moments, void* stream) {
  SC_CHECK_ARG(moments && order >= 1 && n_probe >= 1 && lambda_max > 0.0, "bad arguments");
  Ranks R;
  SC_TRY(ranks_of(ds, nheld, &R));
  std::vector<double> mu;
  SC_TRY(dist_moments(R, lambda_max, order, n_probe, seed, row0, mu, static_cast<cudaStream_t>(stream)));
  std::memcpy(moments, mu.data(), sizeof(double) * mu.size());
  return SC_OK;
}

int sc_dist_estimate_lambda_k(sc_dist* const* ds, int nheld, int k, double lambda_max, int order, int jackson,
                              int n_probe, uint64_t seed, const int64_t* row0, int max_iter, double rtol,
                              double* lambda_k, double* count_k, void* stream) {
  SC_CHECK_ARG(lambda_k && count_k && k >= 1 && max_iter >= 1 && rtol > 0.0, "bad arguments");
  std::vector<double> mu((size_t)2 * order + 1);
  SC_TRY(sc_dist_cheb_moments(ds, nheld, lambda_max, order, n_probe, seed, row0, mu.data(), stream));
  return lambda_k_dichotomy(mu.data(), order, k, lambda_max, jackson != 0, max_iter, rtol, lambda_k, count_k);
}

int sc_dist_kmeans(sc_comm* const* comms, int nheld, const float* const* F, const int64_t* n_local, int d, int k,
                   int restarts, int max_iter, uint64_t seed, const double* uniforms, int32_t* const* labels,
                   double* centroids, double* inertia, int* iters, int* best_restart, void* stream) {
  SC_CHECK_ARG(comms && nheld >= 1 && F && n_local && labels, "null argument");
  SC_CHECK_ARG(d >= 1 && k >= 1 && restarts >= 1 && max_iter >= 1, "bad arguments");
  const int world = comms[0]->world;
  SC_CHECK_ARG(nheld == 1 || nheld == world, "hold one rank or all ranks of the partition");
  SC_CHECK_ARG(world <= kP2PMaxWorld, "world <= 8");
  for (int r = 0; r < nheld; ++r) {
    SC_CHECK_ARG(comms[r] && comms[r]->world == world && (nheld == 1 || comms[r]->rank == r),
                 "communicators must be ranks 0..world-1 in order");
    SC_CHECK_ARG(n_local[r] >= 1 && F[r] && labels[r] && is_device_ptr(F[r]) && is_device_ptr(labels[r]),
                 "every rank needs >= 1 row; device features and labels required");
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // the ranks' row counts -> each rank's global offset (rank-major point order)
  std::vector<int64_t> counts(world, 0);
  if (nheld == world) {
    for (int r = 0; r < world; ++r) counts[r] = n_local[r];
  } else if (world > 1) {
    SC_CHECK_ARG(comms[0]->comm, "a multi-rank communicator without NCCL cannot run one held rank");
    DevBuf cbuf;
    SC_TRY(cbuf.ensure(sizeof(int64_t) * world));
    SC_CUDA_TRY(cudaMemsetAsync(cbuf.ptr, 0, sizeof(int64_t) * world, s));
    SC_CUDA_TRY(cudaMemcpyAsync(cbuf.as<int64_t>() + comms[0]->rank, n_local, sizeof(int64_t),
                                cudaMemcpyHostToDevice, s));
    SC_NCCL_TRY(ncclAllReduce(cbuf.ptr, cbuf.ptr, world, ncclInt64, ncclSum, comms[0]->comm, s));
    SC_CUDA_TRY(cudaMemcpyAsync(counts.data(), cbuf.ptr, sizeof(int64_t) * world, cudaMemcpyDeviceToHost, s));
    SC_CUDA_TRY(cudaStreamSynchronize(s));
  } else {
    counts[0] = n_local[0];
  }
  std::vector<int64_t> off(world + 1, 0);
  for (int r = 0; r < world; ++r) off[r + 1] = off[r] + counts[r];
  SC_CHECK_ARG(off[world] < (int64_t(1) << 25), "n must be < 2^25 for the exact centroid accumulator");
  std::vector<double> u;
  const double* uh = nullptr;
  if (uniforms) {
    u.assign(uniforms, uniforms + (size_t)restarts * k);
    uh = u.data();
  }
  std::vector<double> C((size_t)k * d);
  double in = 0.0;
  int it = 0, best = 0;
  if (nheld == 1) {
    sc_comm* c = comms[0];
    NcclColl coll(c->comm, c->rank, world);
    SC_TRY(kmeans_run_dist(F[0], n_local[0], off[c->rank], off[world], d, k, restarts, max_iter, seed, uh, labels[0],
                           C.data(), &in, &it, &best, &coll, s));
  } else {
    // emulation: one host thread and stream per rank
    LocalGroup grp(world);
    std::vector<int> rcs(world, SC_OK);
    std::vector<std::string> msgs(world);
    std::vector<double> ins(world);
    std::vector<int> its(world), bests(world);
    std::vector<std::vector<double>> Cs(world, std::vector<double>((size_t)k * d));
    int dev = 0;
    cudaGetDevice(&dev);
    SC_CUDA_TRY(cudaStreamSynchronize(s));
    std::vector<std::thread> th;
    for (int r = 0; r < world; ++r) {
      th.emplace_back([&, r]() {
        cudaSetDevice(dev);
        cudaStream_t rs = nullptr;
        int rc = cudaStreamCreateWithFlags(&rs, cudaStreamNonBlocking) == cudaSuccess ? SC_OK : SC_ERR_CUDA;
        LocalColl coll(&grp, r);
        if (rc == SC_OK)
          rc = kmeans_run_dist(F[r], n_local[r], off[r], off[world], d, k, restarts, max_iter, seed, uh, labels[r],
                               Cs[r].data(), &ins[r], &its[r], &bests[r], &coll, rs);
        if (rc != SC_OK) {
          rcs[r] = rc;
          msgs[r] = sc_last_error();
          grp.fail_all();
        }
        if (rs) {
          cudaStreamSynchronize(rs);
          cudaStreamDestroy(rs);
        }
      });
    }
    for (auto& t : th) t.join();
    for (int r = 0; r < world; ++r)
      if (rcs[r] != SC_OK) return fail(rcs[r], "sc_dist_kmeans rank " + std::to_string(r) + ": " + msgs[r]);
    for (int r = 1; r < world; ++r)
      if (Cs[r] != Cs[0] || ins[r] != ins[0] || its[r] != its[0] || bests[r] != bests[0])
        return fail(SC_ERR_STATE, "sc_dist_kmeans: ranks disagree on the result");
    C = Cs[0];
    in = ins[0];
    it = its[0];
    best = bests[0];
  }
  if (centroids) std::memcpy(centroids, C.data(), sizeof(double) * C.size());
  if (inertia) *inertia = in;
  if (iters) *iters = it;
  if (best_restart) *best_restart = best;
  return SC_OK;
}

}  // extern "C"
