// tc_accum_test.cu — is tcgen05 fp32 accumulation unbiased?  D[128×64] = Σ_k A·B over K = 4096 (256 MMAs of
// K=16) with all-positive bf16 operands; the mean signed error vs the exact fp64 sum reveals truncation
// (systematically negative) versus round-to-nearest (mean ≈ 0).
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

__global__ void accum_kernel(const float* A, const float* B, float* D, int K) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = sm;              // 128 rows × 64 K (one chunk) bf16
  uint8_t* sB = sm + 16384;      // 64 rows × 64 K
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (threadIdx.x < 32) tmem_alloc<64>(&tbase);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tbase;
  const uint32_t id = idesc(FMT_BF16, FMT_BF16, 128, 64, 0, 0);
  for (int k0 = 0; k0 < K; k0 += 64) {
    for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) {
      int r = i / 64, k = i % 64;
      *(__nv_bfloat16*)(sA + sw128(r, k * 2)) = __float2bfloat16_rn(A[(size_t)r * K + k0 + k]);
      if (r < 64) *(__nv_bfloat16*)(sB + sw128(r, k * 2)) = __float2bfloat16_rn(B[(size_t)r * K + k0 + k]);
    }
    fence_proxy_async_smem();
    tc_fence_before(); __syncthreads(); tc_fence_after();
    if (threadIdx.x == 0) {
      for (int kk = 0; kk < 4; ++kk)
        mma_bf16(tmem, smem_desc_sw128(smem_u32(sA) + kk * 32, 16, 1024), smem_desc_sw128(smem_u32(sB) + kk * 32, 16, 1024),
                 id, (k0 | kk) != 0);
      mma_commit(&bar);
    }
    mbar_wait(&bar, (k0 / 64) & 1);
    tc_fence_after();
    __syncthreads();
  }
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int c0 = 0; c0 < 64; c0 += 16) {
    float v[16];
    tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
    for (int j = 0; j < 16; ++j) D[(warp * 32 + lane) * 64 + c0 + j] = v[j];
  }
  tc_fence_before(); __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<64>(tmem);
}

int main() {
  const int K = 4096;
  std::vector<float> A(128 * K), B(64 * K), D(128 * 64);
  srand(7);
  auto bf = [](float x) { return __bfloat162float(__float2bfloat16_rn(x)); };
  for (auto& v : A) v = bf(0.5f + rand() / (float)RAND_MAX);
  for (auto& v : B) v = bf(0.5f + rand() / (float)RAND_MAX);
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(accum_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
  accum_kernel<<<1, 128, 40 * 1024>>>(dA, dB, dD, K);
  printf("kernel: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  double mean = 0, mabs = 0, mfp32 = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 64; ++n) {
      double ex = 0; float f32 = 0.f;
      for (int k = 0; k < K; ++k) { ex += (double)A[m * K + k] * B[n * K + k]; f32 += A[m * K + k] * B[n * K + k]; }
      double rel = (D[m * 64 + n] - ex) / ex;
      mean += rel; mabs += fabs(rel); mfp32 += (f32 - ex) / ex;
    }
  printf("tcgen05 fp32 accumulation over K=%d: mean rel err %.3e, mean |rel err| %.3e  (sequential fp32 FMA RN: mean %.3e)\n",
         K, mean / 8192, mabs / 8192, mfp32 / 8192);
  printf("truncation would give a mean near -%.1e; round-to-nearest near 0\n", 0.5 * 256 * pow(2.0, -24));
  return 0;
}
