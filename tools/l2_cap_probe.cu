// Micro-benchmark (tooling, not product): the L2 -> SM throughput ceiling of this B200 in bytes
// per SM-clock cycle, the figure /opt/skills/guides/B300_MICROARCH.md calls the "LTS throughput
// cap" (~6100-6300 B/cycle on B300, whatever the access path).  Every SM reads an L2-resident
// buffer (8..96 MB, ld.global.cg: no L1) over and over, (a) sequentially, (b) as random 128-byte
// rows (the Chebyshev SpMM's gather: 8 lanes x 16 B per row).  The SM clock is measured inside the
// run (clock64 against globaltimer), so the result is per cycle at the clock the GPU really ran.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_cap_probe tools/l2_cap_probe.cu
//   ./l2_cap_probe [col_idx.int32 table_rows] > gpurun_out/l2_cap_probe.txt
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <random>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ float4 ldcg(const float4* p) {
  float4 v;
  asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// clk[0..1]: clock64 / globaltimer at the start of block 0, clk[2..3] at its end
template <int U>
__global__ void __launch_bounds__(512) seq_read(const float4* __restrict__ buf, int64_t nvec, int reps, float4* out,
                                                unsigned long long* clk) {
  if (blockIdx.x == 0 && threadIdx.x == 0) { clk[0] = clock64(); clk[1] = gtimer(); }
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  float4 acc = make_float4(0, 0, 0, 0);
  for (int r = 0; r < reps; ++r) {
    // every thread block starts at a different offset so the SMs do not march in lock step
    const int64_t off = ((int64_t)blockIdx.x * 7919 * 512) % nvec;
    for (int64_t i = tid; i < nvec; i += nth * U) {
      float4 g[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        int64_t j = i + u * nth;
        const bool in = j < nvec;
        j += off;
        j = j >= nvec ? j - nvec : j;
        g[u] = in ? ldcg(buf + j) : make_float4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) { acc.x += g[u].x; acc.y += g[u].y; acc.z += g[u].z; acc.w += g[u].w; }
    }
  }
  if (acc.x == 1234.5f) out[threadIdx.x] = acc;
  if (blockIdx.x == 0 && threadIdx.x == 0) { clk[2] = clock64(); clk[3] = gtimer(); }
}

// random 128-byte rows: 8 lanes per row, EB rows in flight per lane group
template <int EB>
__global__ void __launch_bounds__(512) row_gather(const float4* __restrict__ T, const int32_t* __restrict__ idx,
                                                  int64_t nedges, float4* out, unsigned long long* clk) {
  if (blockIdx.x == 0 && threadIdx.x == 0) { clk[0] = clock64(); clk[1] = gtimer(); }
  const int lane = threadIdx.x & 31, sub = lane >> 3, sl = lane & 7;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (gridDim.x * (int64_t)blockDim.x) >> 5;
  float4 acc = make_float4(0, 0, 0, 0);
  for (int64_t base = (warp * 4 + sub) * EB; base + EB <= nedges; base += nwarps * 4 * EB) {
    int k[EB];
#pragma unroll
    for (int e = 0; e < EB; ++e) k[e] = __ldg(idx + base + e);
    float4 g[EB];
#pragma unroll
    for (int e = 0; e < EB; ++e) g[e] = ldcg(T + (int64_t)k[e] * 8 + sl);
#pragma unroll
    for (int e = 0; e < EB; ++e) { acc.x += g[e].x; acc.y += g[e].y; acc.z += g[e].z; acc.w += g[e].w; }
  }
  if (acc.x == 1234.5f) out[threadIdx.x] = acc;
  if (blockIdx.x == 0 && threadIdx.x == 0) { clk[2] = clock64(); clk[3] = gtimer(); }
}

int main(int argc, char** argv) {
  int dev = 0, sms = 0;
  CK(cudaSetDevice(dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  float4 *buf, *out;
  unsigned long long* clk;
  const size_t maxb = 256ull << 20;
  CK(cudaMalloc(&buf, maxb));
  CK(cudaMemset(buf, 0, maxb));
  CK(cudaMalloc(&out, 1 << 16));
  CK(cudaMalloc(&clk, 64));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  printf("# L2 -> SM throughput, %d SMs; B/cycle uses the SM clock measured in the run (clock64 / globaltimer)\n", sms);
  printf("# kind, MB, blocks/SM, in flight/thread, GB/s, SM MHz, B/cycle\n");
  auto report = [&](const char* kind, size_t mb, int bps, int u, double bytes, float ms) {
    unsigned long long h[4];
    cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
    const double mhz = (double)(h[2] - h[0]) / (double)(h[3] - h[1]) * 1e3;
    const double gbs = bytes / (ms * 1e-3) / 1e9;
    printf("%s, %zu, %d, %d, %.0f, %.0f, %.0f\n", kind, mb, bps, u, gbs, mhz, gbs * 1e9 / (mhz * 1e6));
    fflush(stdout);
  };
  for (size_t mb : {8, 16, 32, 48, 64, 96, 128, 256}) {
    const int64_t nvec = (int64_t)(mb << 20) / 16;
    for (int bps : {2, 4}) {
      const int reps = mb <= 64 ? 40 : 10;
      seq_read<8><<<sms * bps, 512>>>(buf, nvec, 2, out, clk);   // warm the L2
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(e0));
      seq_read<8><<<sms * bps, 512>>>(buf, nvec, reps, out, clk);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      report("sequential", mb, bps, 8, (double)(mb << 20) * reps, ms);
    }
  }
  if (argc >= 3) {
    // a real index stream (int32 file: a graph's CSR column indices in row order) gathered as
    // 128-byte rows from a table of argv[2] rows: the SpMM's gathers without any of its streams
    FILE* f = fopen(argv[1], "rb");
    if (!f) { printf("cannot open %s\n", argv[1]); return 1; }
    fseek(f, 0, SEEK_END);
    const int64_t ne = ftell(f) / 4;
    fseek(f, 0, SEEK_SET);
    std::vector<int32_t> hi(ne);
    if ((int64_t)fread(hi.data(), 4, ne, f) != ne) { printf("short read\n"); return 1; }
    fclose(f);
    const int64_t rows = atoll(argv[2]);
    if (rows * 128 > (int64_t)maxb) { printf("table too large\n"); return 1; }
    int32_t* di;
    CK(cudaMalloc(&di, ne * 4));
    CK(cudaMemcpy(di, hi.data(), ne * 4, cudaMemcpyHostToDevice));
    for (int bps : {2, 4}) {
      row_gather<4><<<sms * bps, 512>>>(buf, di, ne, out, clk);
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(e0));
      for (int r = 0; r < 5; ++r) row_gather<4><<<sms * bps, 512>>>(buf, di, ne, out, clk);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      report("graph-rows128B", (size_t)(rows * 128 >> 20), bps, 4, (double)ne * 128 * 5, ms);
    }
    CK(cudaFree(di));
  }
  // random 128-byte rows from tables of 16..256 MB
  const int64_t nedges = 200ll * 1000 * 1000;
  int32_t* idx;
  CK(cudaMalloc(&idx, nedges * 4));
  std::vector<int32_t> h(nedges);
  for (size_t mb : {16, 32, 64, 96, 128, 256}) {
    const int64_t rows = (int64_t)(mb << 20) / 128;
    std::mt19937_64 rng(7);
    for (auto& v : h) v = (int32_t)(rng() % rows);
    CK(cudaMemcpy(idx, h.data(), nedges * 4, cudaMemcpyHostToDevice));
    for (int bps : {2, 4}) {
      row_gather<4><<<sms * bps, 512>>>(buf, idx, nedges / 4, out, clk);
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(e0));
      row_gather<4><<<sms * bps, 512>>>(buf, idx, nedges, out, clk);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      report("rows128B", mb, bps, 4, (double)nedges * 128, ms);
    }
  }
  return 0;
}
