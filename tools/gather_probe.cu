// Micro-benchmark (tooling, not product): bandwidth of random row gathers on this B200,
// the access pattern of the Chebyshev SpMM.  For each (row bytes, table size, loads in
// flight per lane) it gathers rows T[idx[e]] for a random index stream idx (int32, read
// sequentially like CSR column indices) and reports gathered GB/s.  Also a streaming copy.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_probe tools/gather_probe.cu
//   ./gather_probe > gpurun_out/gather_probe.txt
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

// VPR lanes per row (16 B each), rows per warp-instruction = 32 / VPR; EB loads in flight per lane
template <int VPR, int EB>
__global__ void __launch_bounds__(512) gather(const float4* __restrict__ T, int64_t rows_ld_vec,
                                              const int32_t* __restrict__ idx, int64_t nedges, float4* __restrict__ out) {
  constexpr int RPW = 32 / VPR;
  const int lane = threadIdx.x & 31, sub = lane / VPR, sl = lane % VPR;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (gridDim.x * (int64_t)blockDim.x) >> 5;
  float4 acc = make_float4(0, 0, 0, 0);
  // each warp-row-group consumes EB consecutive edges per row slot
  for (int64_t base = (warp * RPW + sub) * EB; base < nedges; base += nwarps * RPW * EB) {
    int k[EB];
#pragma unroll
    for (int e = 0; e < EB; ++e) k[e] = (base + e < nedges) ? __ldg(idx + base + e) : 0;
    float4 g[EB];
#pragma unroll
    for (int e = 0; e < EB; ++e) g[e] = __ldg(T + (int64_t)k[e] * rows_ld_vec + sl);
#pragma unroll
    for (int e = 0; e < EB; ++e) { acc.x += g[e].x; acc.y += g[e].y; acc.z += g[e].z; acc.w += g[e].w; }
  }
  if (acc.x == 1234.5f) out[threadIdx.x] = acc;   // keep the loads alive
}

__global__ void copyk(const float4* __restrict__ a, float4* __restrict__ b, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) b[i] = a[i];
}

template <int VPR, int EB>
int run(const float4* T, int64_t nrows, const int32_t* idx, int64_t nedges, float4* out, int sms, const char* tag) {
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gather<VPR, EB>, 512, 0);
  const int grid = sms * occ;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  gather<VPR, EB><<<grid, 512>>>(T, VPR, idx, nedges, out);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) gather<VPR, EB><<<grid, 512>>>(T, VPR, idx, nedges, out);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double bytes = (double)nedges * VPR * 16 * reps;
  printf("%-10s row=%4dB table=%7.1fMB EB=%2d occ=%d : %8.1f GB/s gathered (%.3f ms/pass, %.2f Gedge/s)\n", tag, VPR * 16,
         nrows * VPR * 16 / 1e6, EB, occ, bytes / (ms / 1e3) / 1e9, ms / reps, nedges * reps / (ms / 1e3) / 1e9);
  return 0;
}

int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t nedges = 20'000'000;
  std::vector<int32_t> h(nedges);
  float4 *T, *out, *B;
  int32_t* idx;
  const size_t maxT = (size_t)1 << 30;
  CK(cudaMalloc(&T, maxT)); CK(cudaMalloc(&B, maxT)); CK(cudaMalloc(&out, 1 << 20)); CK(cudaMalloc(&idx, nedges * 4));
  CK(cudaMemset(T, 0, maxT));
  // streaming copy (read + write bytes)
  {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int64_t n = maxT / 16;
    copyk<<<sms * 8, 512>>>(T, B, n);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) copyk<<<sms * 8, 512>>>(T, B, n);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("copy 1 GiB: %.1f GB/s (read+write)\n", 2.0 * maxT * 5 / (ms / 1e3) / 1e9);
  }
  std::mt19937_64 rng(1);
  for (double mb : {16.0, 32.0, 64.0, 96.0, 128.0, 256.0, 1024.0}) {
    for (int rb : {64, 128, 256}) {
      const int64_t nrows = (int64_t)(mb * 1e6 / rb);
      if (nrows * rb > (int64_t)maxT) continue;
      std::uniform_int_distribution<int64_t> d(0, nrows - 1);
      for (auto& v : h) v = (int32_t)d(rng);
      CK(cudaMemcpy(idx, h.data(), nedges * 4, cudaMemcpyHostToDevice));
      char tag[32]; snprintf(tag, sizeof tag, "rand");
      if (rb == 64) { run<4, 8>(T, nrows, idx, nedges, out, sms, tag); run<4, 16>(T, nrows, idx, nedges, out, sms, tag); }
      if (rb == 128) { run<8, 4>(T, nrows, idx, nedges, out, sms, tag); run<8, 8>(T, nrows, idx, nedges, out, sms, tag); run<8, 16>(T, nrows, idx, nedges, out, sms, tag); }
      if (rb == 256) { run<16, 4>(T, nrows, idx, nedges, out, sms, tag); run<16, 8>(T, nrows, idx, nedges, out, sms, tag); run<16, 16>(T, nrows, idx, nedges, out, sms, tag); }
    }
  }
  return 0;
}
