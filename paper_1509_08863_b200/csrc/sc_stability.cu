// Stability measure gamma(k) (§4.3, Eq.(11)) reusing the
// fused Chebyshev step kernel.
//
// For every k in [k_min, k_max] the paper runs the accelerated algorithm J times
// with J realisations of the random signals and averages the ARI over all pairs
// of the J clusterings.  Only the cut lambda~_k depends on k; the Chebyshev
// terms T_m(L~) X_j of one realisation X_j do not.  So each realisation runs the
// recurrence once (p fused steps, y_mode 0, every T_m kept in HBM: (p+1) N R
// floats) and one streaming kernel forms the filtered block of every cut,
//     Y_k = sum_m d_{k,m} T_m      (d_k: Chebyshev coefficients of h_{lambda~_k}),
// reading the T_m stack once per group of 8 cuts.  k-means and the ARI are the
// library's own kernels.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "sc_internal.cuh"

namespace sc {
namespace {

bool env_resident() {
  const char* v = std::getenv("SC_RESIDENT");
  return !(v && std::atoi(v) == 0);
}

constexpr int kKG = 8;   // cuts formed per pass over the T_m stack

// Y[g][i*R + q] = sum_m D[g][m] * T[m][i*ld + q]  for the kg cuts of this pass
__global__ void combine_cuts_kernel(const float* __restrict__ Tall, int64_t slot, int nterms, int64_t n, int R,
                                    int ld, const float* __restrict__ D, int kg, float* __restrict__ Y,
                                    int64_t ystride) {
  extern __shared__ float sD[];   // [kKG][nterms]
  for (int e = threadIdx.x; e < kg * nterms; e += blockDim.x) sD[e] = D[e];
  __syncthreads();
  const int64_t total = n * R;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / R;
    const int q = static_cast<int>(idx - i * R);
    const float* t = Tall + i * ld + q;
    float acc[kKG];
#pragma unroll
    for (int c = 0; c < kKG; ++c) acc[c] = 0.f;
    for (int m = 0; m < nterms; ++m) {
      const float v = __ldg(t + (int64_t)m * slot);
#pragma unroll
      for (int c = 0; c < kKG; ++c)
        if (c < kg) acc[c] = fmaf(sD[c * nterms + m], v, acc[c]);
    }
#pragma unroll
    for (int c = 0; c < kKG; ++c)
      if (c < kg) Y[(int64_t)c * ystride + idx] = acc[c];
  }
}

__global__ void pad_copy_kernel(const float* __restrict__ src, int64_t n, int R, float* __restrict__ dst, int ld) {
  const int64_t total = n * ld;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / ld;
    const int q = static_cast<int>(idx - i * ld);
    dst[idx] = q < R ? src[i * R + q] : 0.f;
  }
}

// ARI of every replicate pair of every cut (§4.3 Eq.(11); same formula and
// degenerate-case rule as ari_dev / the oracle, R9): block = one pair (cut c,
// replicates a < b), contingency table of the two labelings in shared memory (labels of cut
// c are in [0, k_min + c)), then the pair-count sums in fp64 by one thread.
__global__ void pair_ari_kernel(const int32_t* __restrict__ labels, int64_t n, int J, int k_min,
                                const int2* __restrict__ pairs_of, const int* __restrict__ cut_of,
                                double* __restrict__ out) {
  extern __shared__ unsigned tab[];
  const int pid = blockIdx.x;
  const int c = cut_of[pid];
  const int2 ab = pairs_of[pid];
  const int k = k_min + c;
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) tab[e] = 0u;
  __syncthreads();
  const int32_t* la = labels + ((size_t)c * J + ab.x) * n;
  const int32_t* lb = labels + ((size_t)c * J + ab.y) * n;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) atomicAdd(&tab[la[i] * k + lb[i]], 1u);
  __syncthreads();
  if (threadIdx.x == 0) {
    auto c2 = [](double x) { return x * (x - 1.0) / 2.0; };
    double sum_ij = 0.0, sa = 0.0, sb = 0.0;
    int64_t nnz = 0;
    int nra = 0, ncb = 0;
    for (int i = 0; i < k; ++i) {
      double ra = 0.0;
      for (int j = 0; j < k; ++j) {
        const double v = (double)tab[i * k + j];
        if (v > 0) ++nnz;
        sum_ij += c2(v);
        ra += v;
      }
      sa += c2(ra);
      nra += ra > 0;
    }
    for (int j = 0; j < k; ++j) {
      double cb = 0.0;
      for (int i = 0; i < k; ++i) cb += (double)tab[i * k + j];
      sb += c2(cb);
      ncb += cb > 0;
    }
    const double expected = n > 1 ? sa * sb / c2((double)n) : 0.0;
    const double denom = 0.5 * (sa + sb) - expected;
    out[pid] = denom == 0.0 ? ((nra == ncb && nnz == nra) ? 1.0 : 0.0) : (sum_ij - expected) / denom;
  }
}

}  // namespace

int stability_scan(sc_graph* g, int k_min, int k_max, int J, int R, int order, bool jackson, int n_probe,
                   uint64_t seed, int restarts, int max_iter, double lambda_max, const double* lambda_k_in,
                   double* gamma, double* lambda_k_out, int32_t* labels_dev, cudaStream_t s) {
  const int64_t n = g->n_rows;
  const int K = k_max - k_min + 1;
  // 1. spectral bounds
  if (!(lambda_max > 0.0)) {
    double theta = 0.0;
    SC_TRY(lanczos_lambda_max(g, 60, seed ^ 0x1a2b3c4dULL, &theta, s));
    const double gersh = 2.0 * g->max_strength;
    lambda_max = 1.01 * theta;
    if (!(lambda_max > 0.0) || lambda_max > gersh) lambda_max = gersh;
    if (!(lambda_max > 0.0)) lambda_max = 1.0;
  }
  std::vector<double> lk(K);
  if (lambda_k_in) {
    std::copy(lambda_k_in, lambda_k_in + K, lk.begin());
  } else {
    // one moments pass serves the dichotomy of every k
    DevBuf probes;
    SC_TRY(probes.ensure(sizeof(double) * n * n_probe));
    SC_TRY(random_signals<double>(n, n_probe, 0, seed ^ 0x5e5e5e5eULL, 2, 1.0 / n_probe, probes.as<double>(), s));
    std::vector<double> mu;
    SC_TRY(cheb_moments(g, lambda_max, order, n_probe, probes.as<double>(), mu, s));
    for (int c = 0; c < K; ++c) {
      double ck = 0.0;
      SC_TRY(lambda_k_dichotomy(mu.data(), order, k_min + c, lambda_max, true, 40, 1e-4, &lk[c], &ck));
    }
  }
  if (lambda_k_out) std::copy(lk.begin(), lk.end(), lambda_k_out);

  // 2. coefficients of every cut, fp32 (the precision the fused filter applies them in)
  const int nterms = order + 1;
  std::vector<float> D((size_t)K * nterms);
  std::vector<double> d(nterms);
  for (int c = 0; c < K; ++c) {
    cheby_lowpass_coeffs(lk[c], lambda_max, order, jackson, d.data());
    for (int m = 0; m < nterms; ++m) D[(size_t)c * nterms + m] = static_cast<float>(d[m]);
  }
  DevBuf dD;
  SC_TRY(dD.ensure(sizeof(float) * D.size()));
  SC_CUDA_TRY(cudaMemcpyAsync(dD.ptr, D.data(), sizeof(float) * D.size(), cudaMemcpyHostToDevice, s));

  // 3. buffers: T stack (ld = R rounded up to 4), the features of every cut for a group of
  // replicates (as many as fit half of the free memory), signals
  const int ld = (R + 3) / 4 * 4;
  const int64_t slot = n * ld;
  const size_t per_rep = sizeof(float) * (size_t)K * n * R;
  size_t free_b = 0, total_b = 0;
  cudaMemGetInfo(&free_b, &total_b);
  const size_t tall_bytes = sizeof(float) * (size_t)slot * nterms;
  const size_t budget = free_b > tall_bytes ? (free_b - tall_bytes) / 2 : 0;
  const int Jg = (int)std::max<size_t>(1, std::min<size_t>((size_t)J, budget / std::max<size_t>(per_rep, 1)));
  DevBuf tall, yall, sig;
  SC_TRY(tall.ensure(tall_bytes));
  SC_TRY(yall.ensure(per_rep * Jg));
  if (ld != R) SC_TRY(sig.ensure(sizeof(float) * n * R));
  float* T = tall.as<float>();
  const std::vector<int> chunks = chunk_widths<float>(ld, n);
  const int grid = g->num_sms * 8;
  int dev = 0;
  cudaGetDevice(&dev);

  const bool trace = std::getenv("SC_STABILITY_TRACE") != nullptr;
  auto now = [] { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
  double t_filter = 0.0, t_kmeans = 0.0, t_mark = now();
  for (int j0 = 0; j0 < J; j0 += Jg) {
    const int jn = std::min(Jg, J - j0);
    if (trace) t_mark = now();
    // 3a. recurrence + every cut's features for replicates j0 .. j0+jn-1 (stream s)
    for (int jj = 0; jj < jn; ++jj) {
      const uint64_t sj = seed + (uint64_t)(j0 + jj);
      // T_0 = X_j (§4.1 step 4: N(0, 1/R) entries)
      if (ld == R) {
        SC_TRY(random_signals<float>(n, R, 0, sj, 0, 1.0 / R, T, s));
      } else {
        SC_TRY(random_signals<float>(n, R, 0, sj, 0, 1.0 / R, sig.as<float>(), s));
        pad_copy_kernel<<<grid, 256, 0, s>>>(sig.as<float>(), n, R, T, ld);
        SC_CUDA_TRY(cudaGetLastError());
      }
      // T_{m+1} = 2 L~ T_m - T_{m-1}  (T_1 = L~ T_0), every term kept: one cooperative launch
      // per column chunk when the CSR fits shared memory (resident kernel, stack mode), else
      // one streaming launch per step and chunk
      bool resident = env_resident();
      if (resident) {
        int col0 = 0;
        for (int w : chunks) {
          bool ok = false;
          SC_TRY(resident_filter<float>(g, nullptr, order, lambda_max, w, T + col0, ld, nullptr, 0, nullptr, nullptr, s,
                                        &ok, T + col0, slot));
          if (!ok) { resident = false; break; }
          col0 += w;
        }
        // (a graph that fits does so for every chunk width of the plan; if the first chunk
        // did not, nothing was launched)
      }
      for (int st = 0; st < order && !resident; ++st) {
        int col0 = 0;
        for (int w : chunks) {
          StepParams p{};
          p.row_begin = 0;
          p.row_end = n;
          p.width = w;
          p.total_width = ld;
          p.tcur = T + (size_t)st * slot + col0;
          p.ld_cur = ld;
          p.tprev = st == 0 ? nullptr : (const void*)(T + (size_t)(st - 1) * slot + col0);
          p.ld_prev = ld;
          p.tnext = T + (size_t)(st + 1) * slot + col0;
          p.ld_next = ld;
          p.a = (st == 0 ? 2.0 : 4.0) / lambda_max;
          p.b_cur = st == 0 ? -1.0 : -2.0;
          p.b_prev = st == 0 ? 0.0 : -1.0;
          p.y_mode = 0;
          SC_TRY(launch_step<float>(g, p, s));
          col0 += w;
        }
      }
      // Y_k for every cut
      float* yj = yall.as<float>() + (size_t)jj * K * n * R;
      for (int c0 = 0; c0 < K; c0 += kKG) {
        const int kg = std::min(kKG, K - c0);
        combine_cuts_kernel<<<grid, 256, sizeof(float) * kg * nterms, s>>>(
            T, slot, nterms, n, R, ld, dD.as<float>() + (size_t)c0 * nterms, kg, yj + (size_t)c0 * n * R, n * R);
        SC_CUDA_TRY(cudaGetLastError());
      }
    }
    if (trace) { SC_CUDA_TRY(cudaStreamSynchronize(s)); t_filter += now() - t_mark; t_mark = now(); }
    cudaEvent_t ready;
    SC_CUDA_TRY(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    SC_CUDA_TRY(cudaEventRecord(ready, s));
    // 3b. the jn*K k-means problems (§4.1 step 6; replicate seed seed+j) are
    // independent and individually too small to fill the GPU: worker threads, each with its
    // own stream and stream-ordered workspaces, run them concurrently
    const int ntask = jn * K;
    const int nwork = std::min(ntask, std::getenv("SC_STABILITY_WORKERS") ? std::max(1, std::atoi(std::getenv("SC_STABILITY_WORKERS"))) : 8);
    std::atomic<int> next{0};
    std::mutex err_mu;
    int err_code = SC_OK;
    std::string err_msg;
    auto worker = [&]() {
      cudaSetDevice(dev);
      cudaStream_t ws = nullptr;
      if (cudaStreamCreateWithFlags(&ws, cudaStreamNonBlocking) != cudaSuccess ||
          cudaStreamWaitEvent(ws, ready, 0) != cudaSuccess) {
        std::lock_guard<std::mutex> lk(err_mu);
        if (err_code == SC_OK) { err_code = SC_ERR_CUDA; err_msg = "worker stream creation failed"; }
        if (ws) cudaStreamDestroy(ws);
        return;
      }
      for (int t = next++; t < ntask; t = next++) {
        const int jj = t / K, c = t - jj * K;
        const int j = j0 + jj;
        double inertia = 0.0;
        int it = 0, best = 0;
        const int rc = kmeans_run(yall.as<float>() + ((size_t)jj * K + c) * n * R, n, R, k_min + c, restarts,
                                  max_iter, seed + (uint64_t)j, nullptr, labels_dev + ((size_t)c * J + j) * n,
                                  nullptr, &inertia, &it, &best, ws, 4);
        if (rc != SC_OK) {
          std::lock_guard<std::mutex> lk(err_mu);
          if (err_code == SC_OK) { err_code = rc; err_msg = sc_last_error(); }
          break;
        }
      }
      cudaStreamSynchronize(ws);
      cudaStreamDestroy(ws);
    };
    std::vector<std::thread> pool;
    for (int w = 0; w < nwork; ++w) pool.emplace_back(worker);
    for (auto& th : pool) th.join();
    cudaEventDestroy(ready);
    if (err_code != SC_OK) return fail(err_code, "sc_stability k-means worker: " + err_msg);
    if (trace) t_kmeans += now() - t_mark;
  }
  if (trace) t_mark = now();
  // 4. gamma(k) = 2/(J(J-1)) sum_{a<b} ari(C^a, C^b)   (R7): every pair's ARI in one
  // launch when the contingency tables fit shared memory, else pair by pair
  if ((size_t)k_max * k_max * sizeof(unsigned) <= 96 * 1024) {
    std::vector<int2> pr;
    std::vector<int> cut;
    for (int c = 0; c < K; ++c)
      for (int a = 0; a < J; ++a)
        for (int b = a + 1; b < J; ++b) {
          pr.push_back(make_int2(a, b));
          cut.push_back(c);
        }
    const int np = (int)pr.size();
    std::vector<double> aris(np, 0.0);
    if (np) {
      DevBuf dp, dc, da;
      SC_TRY(dp.ensure(sizeof(int2) * np));
      SC_TRY(dc.ensure(sizeof(int) * np));
      SC_TRY(da.ensure(sizeof(double) * np));
      SC_CUDA_TRY(cudaMemcpyAsync(dp.ptr, pr.data(), sizeof(int2) * np, cudaMemcpyHostToDevice, s));
      SC_CUDA_TRY(cudaMemcpyAsync(dc.ptr, cut.data(), sizeof(int) * np, cudaMemcpyHostToDevice, s));
      const int smem = (int)(sizeof(unsigned) * k_max * k_max);
      if (smem > 48 * 1024)
        SC_CUDA_TRY(cudaFuncSetAttribute(pair_ari_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      pair_ari_kernel<<<np, 256, smem, s>>>(labels_dev, n, J, k_min, dp.as<int2>(), dc.as<int>(), da.as<double>());
      SC_CUDA_TRY(cudaGetLastError());
      SC_CUDA_TRY(cudaMemcpyAsync(aris.data(), da.ptr, sizeof(double) * np, cudaMemcpyDeviceToHost, s));
      SC_CUDA_TRY(cudaStreamSynchronize(s));
    }
    int i = 0;
    for (int c = 0; c < K; ++c) {
      double tot = 0.0;
      for (int a = 0; a < J; ++a)
        for (int b = a + 1; b < J; ++b) tot += aris[i++];
      gamma[c] = 2.0 * tot / ((double)J * (J - 1));
    }
  } else {
    for (int c = 0; c < K; ++c) {
      double tot = 0.0;
      for (int a = 0; a < J; ++a)
        for (int b = a + 1; b < J; ++b) {
          double v = 0.0;
          SC_TRY(ari_dev(labels_dev + ((size_t)c * J + a) * n, labels_dev + ((size_t)c * J + b) * n, n, &v, s));
          tot += v;
        }
      gamma[c] = 2.0 * tot / ((double)J * (J - 1));
    }
  }
  if (trace)
    std::fprintf(stderr, "[sc_stability] J=%d groups of %d: recurrence+cuts %.4f s, k-means %.4f s, ARI %.4f s\n", J, Jg,
                 t_filter, t_kmeans, now() - t_mark);
  return SC_OK;
}

}  // namespace sc
