// Probe (tooling): the tcgen05 kind::tf32 mechanics the k-means tensor screen uses --
// K-major no-swizzle shared-memory descriptors, instruction descriptor, TMEM allocation,
// one-thread MMA issue, commit to an mbarrier, tcgen05.ld of the accumulator.
// S[m][n] = sum_k A[m][k] * B[n][k] for A 128 x K, B N x K (tf32-rounded), vs a host fp64
// reference of the same tf32-rounded inputs; prints the max relative error and time.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tcp tools/tc_probe.cu && ./tcp
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>
#include <random>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major, no swizzle: 16-byte chunk (row r, k-chunk j) at ((r % 8) + (r / 8) * SBO + j * LBO) * 16 B
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;   // version (Blackwell)
  return d;                  // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}

__device__ __forceinline__ uint32_t idesc_tf32(int M, int N) {
  return (1u << 4)              // D format F32
         | (2u << 7)            // A format TF32
         | (2u << 10)           // B format TF32
         | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);   // K-major A and B (bits 15, 16 = 0)
}

template <int K, int N>
__global__ void __launch_bounds__(128) tc_kernel(const float* __restrict__ A, const float* __restrict__ B,
                                                 float* __restrict__ S) {
  constexpr int M = 128;
  constexpr int KC = K / 4;   // 16-byte chunks per row
  extern __shared__ __align__(1024) float dsm[];
  float* sA = dsm;
  float* sB = dsm + M * K;
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  // canonical K-major no-swizzle layout: LBO = 128 B (next k-chunk of the same 8 rows),
  // SBO = KC * 128 B (next group of 8 rows)
  for (int i = tid; i < M * KC; i += blockDim.x) {
    const int r = i / KC, j = i % KC;
    const float4 v = *reinterpret_cast<const float4*>(A + r * K + 4 * j);
    float* dst = sA + (((r % 8) + (r / 8) * (8 * KC) + j * 8) * 4);
    float4 t;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(*(uint32_t*)&t.x) : "f"(v.x));
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(*(uint32_t*)&t.y) : "f"(v.y));
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(*(uint32_t*)&t.z) : "f"(v.z));
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(*(uint32_t*)&t.w) : "f"(v.w));
    *reinterpret_cast<float4*>(dst) = t;
  }
  for (int i = tid; i < N * KC; i += blockDim.x) {
    const int r = i / KC, j = i % KC;
    const float4 v = *reinterpret_cast<const float4*>(B + r * K + 4 * j);
    float* dst = sB + (((r % 8) + (r / 8) * (8 * KC) + j * 8) * 4);
    float4 t;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(*(uint32_t*)&t.x) : "f"(v.x));
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(*(uint32_t*)&t.y) : "f"(v.y));
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(*(uint32_t*)&t.z) : "f"(v.z));
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(*(uint32_t*)&t.w) : "f"(v.w));
    *reinterpret_cast<float4*>(dst) = t;
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(N <= 32 ? 32 : N <= 64 ? 64 : N <= 128 ? 128 : 256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic smem writes -> async proxy
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint32_t id = idesc_tf32(M, N);
#pragma unroll
    for (int ks = 0; ks < K / 8; ++ks) {   // one MMA covers K = 8 tf32 (two 16-byte chunks)
      const uint64_t da = umma_desc(smem_u32(sA) + ks * 2 * 128, 128, KC * 128);
      const uint64_t db = umma_desc(smem_u32(sB) + ks * 2 * 128, 128, KC * 128);
      const uint32_t acc = ks > 0;
      asm volatile(
          "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
          "l"(da), "l"(db), "r"(id), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                 : "memory");
  }
  // wait for the MMAs
  asm volatile(
      "{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W;\n}\n" ::"r"(
          smem_u32(&bar))
      : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // row m = tid (TMEM lane), 32 columns per load
  for (int c0 = 0; c0 < N; c0 += 8) {
    uint32_t v[8];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int q = 0; q < 8; ++q) S[tid * N + c0 + q] = __uint_as_float(v[q]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(N <= 32 ? 32 : N <= 64 ? 64 : N <= 128 ? 128 : 256));
}

static float tf32_host(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  u = (u + 0x1000u) & ~0x1FFFu;   // round to nearest (ties away), 10-bit mantissa
  float r;
  memcpy(&r, &u, 4);
  return r;
}

template <int K, int N>
int run() {
  constexpr int M = 128;
  std::mt19937 rng(1);
  std::normal_distribution<float> nd(0.f, 1.f);
  std::vector<float> A(M * K), B(N * K), S(M * N);
  for (auto& v : A) v = nd(rng);
  for (auto& v : B) v = nd(rng);
  float *dA, *dB, *dS;
  CK(cudaMalloc(&dA, A.size() * 4));
  CK(cudaMalloc(&dB, B.size() * 4));
  CK(cudaMalloc(&dS, S.size() * 4));
  CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
  const int smem = (M + N) * K * 4;
  CK(cudaFuncSetAttribute(tc_kernel<K, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  tc_kernel<K, N><<<1, 128, smem>>>(dA, dB, dS);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(S.data(), dS, S.size() * 4, cudaMemcpyDeviceToHost));
  double maxerr = 0, maxref = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double ref = 0, mag = 0;
      for (int k = 0; k < K; ++k) {
        const double p = (double)tf32_host(A[m * K + k]) * (double)tf32_host(B[n * K + k]);
        ref += p;
        mag += fabs(p);
      }
      maxerr = fmax(maxerr, fabs(S[m * N + n] - ref) / mag);
      maxref = fmax(maxref, fabs(ref));
    }
  printf("K=%d N=%d: max |S - ref| / sum|a b| = %.3e (2^-23 = %.3e)  S[0]=%f S[last]=%f\n", K, N, maxerr,
         ldexp(1.0, -23), S[0], S[M * N - 1]);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dS);
  return 0;
}

int main() {
  run<64, 104>();
  run<64, 128>();
  run<96, 200>();
  run<16, 32>();
  return 0;
}
