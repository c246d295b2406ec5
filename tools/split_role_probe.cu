// Micro-benchmark (tooling, not product): one Chebyshev step over a real CSR graph with the
// warps of a CTA split by role -- 12 gather warps (8 lanes per row, 4 loads in flight per lane)
// that only sum the neighbours' rows of T_s and park the row sums in shared memory, 4 epilogue
// warps that stream own / T_{s-1} / Y, apply the recurrence and store -- at 32 registers per
// thread, i.e. 4 CTAs x 512 threads = 2048 threads per SM (the thread count at which
// tools/l2_cap_probe.cu gathers configs[3]'s index stream at 17.5 TB/s).  32-column fp32 chunks
// (128-byte rows), unit weights, no degree sorting, static tiles.  DESIGN.md §0(f).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o split_role_probe tools/split_role_probe.cu
//   ./split_role_probe row_ptr.int64 col_idx.int32 n_rows
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int kGW = 12, kEW = 4, kTR = kGW * 4;   // gather warps, epilogue warps, rows per tile

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n"
               ::"r"(smem_u32(b)), "r"(parity) : "memory");
}

template <int MINB>
__global__ void __launch_bounds__((kGW + kEW) * 32, MINB)
split_step(const float4* __restrict__ Tc, const float4* Tp, float4* Tn, float4* Y, int yflag,
           const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col, int n, float a, float b, float c, int epi) {
  __shared__ __align__(16) float4 S[2][kTR][8];
  __shared__ uint64_t full[2], empty[2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, sub = lane >> 3, sl = lane & 7;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) { mbar_init(&full[i], kGW); mbar_init(&empty[i], kEW); }
  }
  __syncthreads();
  const int ntiles = (n + kTR - 1) / kTR;
  if (warp < kGW) {
    int it = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      const int buf = it & 1;
      if (it >= 2) mbar_wait(&empty[buf], ((it >> 1) - 1) & 1);
      const int rl = warp * 4 + sub, r = t * kTR + rl;
      float4 acc = make_float4(0, 0, 0, 0);
      if (r < n) {
        const int64_t e0 = row_ptr[r], e1 = row_ptr[r + 1];
        for (int64_t e = e0; e < e1; e += 4) {
          int k[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) k[j] = e + j < e1 ? __ldg(col + e + j) : n;   // row n: zeros
          float4 g[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) g[j] = __ldg(Tc + (int64_t)k[j] * 8 + sl);
#pragma unroll
          for (int j = 0; j < 4; ++j) { acc.x += g[j].x; acc.y += g[j].y; acc.z += g[j].z; acc.w += g[j].w; }
        }
      }
      S[buf][rl][sl] = acc;
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[buf]);
    }
  } else {
    const int ew = warp - kGW;
    int it = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      const int buf = it & 1;
      mbar_wait(&full[buf], (it >> 1) & 1);
#pragma unroll 1
      for (int q = 0; q < kTR / (kEW * 4); ++q) {
        const int rl = (q * kEW + ew) * 4 + sub, r = t * kTR + rl;
        if (r < n && epi) {
          const float4 s = S[buf][rl][sl];
          const int64_t o = (int64_t)r * 8 + sl;
          const float4 own = __ldg(Tc + o);
          const float4 prv = Tp[o];
          const float deg = (float)(row_ptr[r + 1] - row_ptr[r]);
          float4 tn;
          tn.x = a * (deg * own.x - s.x) + b * own.x + c * prv.x;
          tn.y = a * (deg * own.y - s.y) + b * own.y + c * prv.y;
          tn.z = a * (deg * own.z - s.z) + b * own.z + c * prv.z;
          tn.w = a * (deg * own.w - s.w) + b * own.w + c * prv.w;
          Tn[o] = tn;
          if (yflag) {
            float4 y = Y[o];
            y.x += 0.1f * prv.x + 0.2f * own.x + 0.3f * tn.x;
            y.y += 0.1f * prv.y + 0.2f * own.y + 0.3f * tn.y;
            y.z += 0.1f * prv.z + 0.2f * own.z + 0.3f * tn.z;
            y.w += 0.1f * prv.w + 0.2f * own.w + 0.3f * tn.w;
            Y[o] = y;
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[buf]);
    }
  }
}

template <int MINB>
int run(const char* tag, float4* const* T, float4* Y, const int64_t* rp, const int32_t* ci, int n, int64_t nnz, int sms, int epi) {
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, split_step<MINB>, (kGW + kEW) * 32, 0));
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, split_step<MINB>));
  const int grid = sms * occ;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int steps = 60;
  for (int rep = 0; rep < 2; ++rep) {
    CK(cudaEventRecord(e0));
    for (int s = 0; s < steps; ++s)
      split_step<MINB><<<grid, (kGW + kEW) * 32>>>(T[s % 2], T[(s + 1) % 2], T[(s + 1) % 2], Y, s % 3 == 2, rp, ci, n,
                                                  1e-3f, -0.5f, -0.25f, epi);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
  }
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  const double us = ms * 1e3 / steps;
  printf("%s: %d regs, %zu B local, %d CTAs/SM (%d threads/SM, %d gathering): %.1f us/step, gathers %.0f GB/s\n", tag,
         fa.numRegs, (size_t)fa.localSizeBytes, occ, occ * (kGW + kEW) * 32, occ * kGW * 32, us, (double)nnz * 128 / us / 1e3);
  return 0;
}

int main(int argc, char** argv) {
  if (argc < 4) { printf("usage: %s row_ptr.int64 col_idx.int32 n\n", argv[0]); return 1; }
  const int n = atoi(argv[3]);
  std::vector<int64_t> rp(n + 1);
  FILE* f = fopen(argv[1], "rb");
  if (!f || fread(rp.data(), 8, n + 1, f) != (size_t)n + 1) { printf("row_ptr read failed\n"); return 1; }
  fclose(f);
  const int64_t nnz = rp[n];
  std::vector<int32_t> ci(nnz);
  f = fopen(argv[2], "rb");
  if (!f || (int64_t)fread(ci.data(), 4, nnz, f) != nnz) { printf("col_idx read failed\n"); return 1; }
  fclose(f);
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  float4 *T[2], *Y;
  int64_t* drp;
  int32_t* dci;
  const size_t tb = (size_t)(n + 1) * 128;
  CK(cudaMalloc(&T[0], tb)); CK(cudaMalloc(&T[1], tb)); CK(cudaMalloc(&Y, tb));
  CK(cudaMemset(T[0], 0, tb)); CK(cudaMemset(T[1], 0, tb)); CK(cudaMemset(Y, 0, tb));
  CK(cudaMalloc(&drp, (n + 1) * 8)); CK(cudaMalloc(&dci, nnz * 4));
  CK(cudaMemcpy(drp, rp.data(), (n + 1) * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dci, ci.data(), nnz * 4, cudaMemcpyHostToDevice));
  printf("# role-split step probe: n = %d, nnz = %lld, 32 fp32 columns\n", n, (long long)nnz);
  if (run<4>("full step, 4 CTAs/SM target", T, Y, drp, dci, n, nnz, sms, 1)) return 1;
  if (run<3>("full step, 3 CTAs/SM target", T, Y, drp, dci, n, nnz, sms, 1)) return 1;
  // the same launches with the epilogue's loads and stores switched off: the gathers alone
  if (run<4>("gathers only, 4 CTAs/SM target", T, Y, drp, dci, n, nnz, sms, 0)) return 1;
  if (run<3>("gathers only, 3 CTAs/SM target", T, Y, drp, dci, n, nnz, sms, 0)) return 1;
  return 0;
}
