// Micro-benchmark (tooling, not product): the random-gather ceiling of the Chebyshev step
// WITH the step's other memory streams running alongside.
//
// One "step" over N rows of width w floats, every row gathering DEG random rows of T_s
// (uniform over N, an ELL index array read sequentially like the kernel's staged CSR), then
// reading its own row of T_s and of T_{s-1}, writing T_{s+1} over T_{s-1}, and -- every third
// step -- reading and writing its row of Y.  Buffers rotate like the recurrence (T_s becomes
// T_{s-1} ...), so L2 sees the same mix as cheb_sell_kernel.  Minimal instruction overhead:
// VPR lanes per row, one 16-byte vector per lane, 4 indices per 16-byte load, NB batches of 4
// gathers in flight.  Variants: "gather" (gathers + index stream only) and "step" (all
// streams).  Prints per-launch time, gathered GB/s and G rows/s.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpl tools/gather_probe_load.cu
//   ./gpl > gpurun_out/gather_probe_load.txt
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int DEG = 20;

template <int VPR, int NB, bool STREAMS>
__global__ void __launch_bounds__(512) step(const float4* __restrict__ Tc, const float4* Tp, float4* Tn,
                                            float4* __restrict__ Y, bool ystep, const int4* __restrict__ idx,
                                            int64_t n) {
  constexpr int RPW = 32 / VPR;
  const int lane = threadIdx.x & 31, sub = lane / VPR, sl = lane % VPR;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (gridDim.x * (int64_t)blockDim.x) >> 5;
  for (int64_t r0 = warp * RPW; r0 < n; r0 += nwarps * RPW) {
    const int64_t row = r0 + sub;
    const bool ok = sub < RPW && row < n;
    const int4* ip = idx + (ok ? row : 0) * (DEG / 4);
    float4 acc = make_float4(0, 0, 0, 0);
    float4 g[NB][4];
    auto issue = [&](int s, int b) {
      const int4 k = __ldg(ip + b);
      g[s][0] = __ldg(Tc + (int64_t)k.x * VPR + sl);
      g[s][1] = __ldg(Tc + (int64_t)k.y * VPR + sl);
      g[s][2] = __ldg(Tc + (int64_t)k.z * VPR + sl);
      g[s][3] = __ldg(Tc + (int64_t)k.w * VPR + sl);
    };
    constexpr int NBAT = DEG / 4;
#pragma unroll
    for (int s = 0; s < NB; ++s) issue(s, s);
#pragma unroll
    for (int b = 0; b < NBAT; ++b) {
      const int s = b % NB;
#pragma unroll
      for (int e = 0; e < 4; ++e) { acc.x += g[s][e].x; acc.y += g[s][e].y; acc.z += g[s][e].z; acc.w += g[s][e].w; }
      if (b + NB < NBAT) issue(s, b + NB);
    }
    if (!ok) continue;
    if (STREAMS) {
      const float4 own = Tc[row * VPR + sl];
      const float4 prv = Tp[row * VPR + sl];
      float4 nx;
      nx.x = 0.1f * (own.x - acc.x) - prv.x; nx.y = 0.1f * (own.y - acc.y) - prv.y;
      nx.z = 0.1f * (own.z - acc.z) - prv.z; nx.w = 0.1f * (own.w - acc.w) - prv.w;
      Tn[row * VPR + sl] = nx;
      if (ystep) {
        float4 y = Y[row * VPR + sl];
        y.x += nx.x; y.y += nx.y; y.z += nx.z; y.w += nx.w;
        Y[row * VPR + sl] = y;
      }
    } else if (acc.x == 1234.5f) {
      Tn[threadIdx.x] = acc;
    }
  }
}

template <int VPR, int NB, bool STREAMS>
int run(int64_t n, const int4* idx, float4* A, float4* B, float4* Y, int sms, const char* tag) {
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, step<VPR, NB, STREAMS>, 512, 0);
  const int grid = sms * occ;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float4* buf[2] = {A, B};
  for (int s = 0; s < 3; ++s)
    step<VPR, NB, STREAMS><<<grid, 512>>>(buf[s & 1], buf[(s + 1) & 1], buf[(s + 1) & 1], Y, s % 3 == 2, idx, n);
  CK(cudaDeviceSynchronize());
  const int reps = 30;
  cudaEventRecord(e0);
  for (int s = 0; s < reps; ++s)
    step<VPR, NB, STREAMS><<<grid, 512>>>(buf[s & 1], buf[(s + 1) & 1], buf[(s + 1) & 1], Y, s % 3 == 2, idx, n);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double per = ms / reps * 1e-3;
  const double rows = (double)n * DEG;
  printf("%-7s row=%4dB table=%6.0fMB NB=%d occ=%d : %8.1f us/step  %8.1f GB/s gathered  %6.1f G rows/s\n", tag,
         VPR * 16, n * VPR * 16 / 1e6, NB, occ, per * 1e6, rows * VPR * 16 / per / 1e9, rows / per / 1e9);
  return 0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t n = 1000000;   // configs[3]'s N
  std::mt19937_64 rng(1);
  std::vector<int32_t> h((size_t)n * DEG);
  for (auto& v : h) v = (int32_t)(rng() % n);
  int4* idx;
  float4 *A, *B, *Y;
  CK(cudaMalloc(&idx, h.size() * 4));
  CK(cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
  const size_t maxb = (size_t)n * 64 * 4;
  CK(cudaMalloc(&A, maxb));
  CK(cudaMalloc(&B, maxb));
  CK(cudaMalloc(&Y, maxb));
  CK(cudaMemset(A, 0, maxb));
  CK(cudaMemset(B, 0, maxb));
  CK(cudaMemset(Y, 0, maxb));
  // w = 16, 32, 64 floats (64, 128, 256-byte rows; 64, 128, 256 MB tables)
  run<4, 1, false>(n, idx, A, B, Y, sms, "gather");
  run<4, 1, true>(n, idx, A, B, Y, sms, "step");
  run<4, 2, false>(n, idx, A, B, Y, sms, "gather");
  run<4, 2, true>(n, idx, A, B, Y, sms, "step");
  run<8, 1, false>(n, idx, A, B, Y, sms, "gather");
  run<8, 1, true>(n, idx, A, B, Y, sms, "step");
  run<8, 2, false>(n, idx, A, B, Y, sms, "gather");
  run<8, 2, true>(n, idx, A, B, Y, sms, "step");
  run<16, 1, false>(n, idx, A, B, Y, sms, "gather");
  run<16, 1, true>(n, idx, A, B, Y, sms, "step");
  run<16, 2, false>(n, idx, A, B, Y, sms, "gather");
  run<16, 2, true>(n, idx, A, B, Y, sms, "step");
  return 0;
}
