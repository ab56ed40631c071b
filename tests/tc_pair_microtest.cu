// tc_pair_microtest.cu — semantics check of the 2-CTA (cta_group::2) UMMA before any kernel relies on it:
// a CTA pair computes D[256][256] = A[256][64]·B[256][64]ᵀ in bf16; CTA r holds A rows [128r, 128r+128) and
// (hypothesis) B rows [128r, 128r+128) at the same shared-memory offsets; only CTA 0 issues the MMAs; each CTA
// reads its 128 rows of D from its own TMEM.  Prints max |D − ref| for the hypothesis.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I<repo> tests/tc_pair_microtest.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_bf16.h>
#include "paper_2109_03709_b200/csrc/tc_util.cuh"

using namespace ppca::tc;

__host__ __device__ inline uint32_t sw128(uint32_t row, uint32_t byte) {
  return (row >> 3) * 1024u + (row & 7u) * 128u + ((((byte >> 4) ^ (row & 7u)) << 4) | (byte & 15u));
}

__device__ __forceinline__ uint32_t ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void csync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

constexpr int M = 256, N = 256, K = 64;

__global__ void __cluster_dims__(2, 1, 1) pair_kernel(const float* A, const float* B, float* D, int bsplit) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const uint32_t r = ctarank();
  uint8_t* sA = smem;                 // 128 rows × 64 K (bf16): 16 KB
  uint8_t* sB = smem + 32 * 1024;     // bsplit: 128 rows of B; else all 256 rows (32 KB)
  const int brows = bsplit ? 128 : 256;
  for (int i = threadIdx.x; i < 128 * K; i += blockDim.x) {
    const int m = i / K, k = i % K;
    *(__nv_bfloat16*)(sA + sw128(m, k * 2)) = __float2bfloat16_rn(A[(r * 128 + m) * K + k]);
  }
  for (int i = threadIdx.x; i < brows * K; i += blockDim.x) {
    const int n = i / K, k = i % K;
    const int gn = bsplit ? r * 128 + n : n;
    *(__nv_bfloat16*)(sB + sw128(n, k * 2)) = __float2bfloat16_rn(B[gn * K + k]);
  }
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "n"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  csync();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  if (r == 0 && threadIdx.x == 0) {
    const uint32_t id = idesc(FMT_BF16, FMT_BF16, M, N, 0, 0);
    for (int k0 = 0; k0 < K; k0 += 16) {
      const uint64_t ad = smem_desc_sw128(smem_u32(sA) + k0 * 2, 16, 1024);
      const uint64_t bd = smem_desc_sw128(smem_u32(sB) + k0 * 2, 16, 1024);
      asm volatile(
          "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
          "l"(ad), "l"(bd), "r"(id), "r"((uint32_t)(k0 > 0)));
    }
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(smem_u32(&bar)), "h"((uint16_t)3) : "memory");
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int row = r * 128 + warp * 32 + lane;
  for (int c0 = 0; c0 < N; c0 += 16) {
    float v[16];
    tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
    for (int j = 0; j < 16; ++j) D[row * N + c0 + j] = v[j];
  }
  tc_fence_before();
  __syncthreads();
  csync();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(256));
}

static float bf16r(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }

int main() {
  std::vector<float> A(M * K), B(N * K), D(M * N);
  srand(7);
  for (auto& v : A) v = rand() / (float)RAND_MAX - 0.5f;
  for (auto& v : B) v = rand() / (float)RAND_MAX - 0.5f;
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  for (int bsplit = 1; bsplit >= 0; --bsplit) {
    cudaMemset(dD, 0, D.size() * 4);
    pair_kernel<<<2, 128, 80 * 1024>>>(dA, dB, dD, bsplit);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("bsplit=%d: CUDA error %s\n", bsplit, cudaGetErrorString(e)); return 1; }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double mx = 0, mx_half = 0, scale = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double ref = 0;
        for (int k = 0; k < K; ++k) ref += (double)bf16r(A[m * K + k]) * bf16r(B[n * K + k]);
        mx = fmax(mx, fabs(D[m * N + n] - ref));
        scale = fmax(scale, fabs(ref));
      }
    printf("cta_group::2 M=256 N=256 K=64, B %s: max|D-ref| = %.3e (scale %.2f)\n",
           bsplit ? "split by N across the pair (128 rows each)" : "whole in each CTA", mx, scale);
    (void)mx_half;
  }
  return 0;
}
