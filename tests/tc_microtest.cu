// tc_microtest.cu — one-tile checks of the tcgen05 building blocks used by pass_tc.cu:
// UMMA smem descriptors (K-major / MN-major, SWIZZLE_128B), instruction descriptors (bf16, tf32),
// TMEM alloc + tcgen05.ld, and how kind::tf32 treats fp32 inputs (truncation vs rounding).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I<repo> tests/tc_microtest.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_bf16.h>
#include "paper_2109_03709_b200/csrc/tc_util.cuh"

using namespace ppca::tc;

// byte offset of (row, byte) in a stack of SW128 atoms (8 rows × 128 B each, 1024 B per atom)
__host__ __device__ inline uint32_t sw128(uint32_t row, uint32_t byte) {
  return (row >> 3) * 1024u + (row & 7u) * 128u + ((((byte >> 4) ^ (row & 7u)) << 4) | (byte & 15u));
}

struct Case {
  int tf32;        // 0 bf16, 1 tf32
  int a_mn, b_mn;  // operand majors
  int M, N, K;
};

// A logical [M][K], B logical [N][K] (fp32 host values; bf16/tf32 conversion on device).
// K-major operand: stored [rows][K] in 128-byte K-blocks (block kb holds K range [kb*E, kb*E+E),
//   E = 128/elt), each block = rows × 128 B of SW128 atoms; block stride = rows*128.
// MN-major operand: stored [K][rows] in 128-byte MN-blocks; block stride = K*128.
__global__ void tc_case_kernel(Case cs, const float* A, const float* B, float* D) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int elt = cs.tf32 ? 4 : 2;
  const int E = 128 / elt;                 // elements per 128-B row
  uint8_t* sA = smem;
  uint8_t* sB = smem + 64 * 1024;
  // ---- fill operands
  for (int i = threadIdx.x; i < cs.M * cs.K; i += blockDim.x) {
    int m = i / cs.K, k = i % cs.K;
    uint32_t off;
    if (!cs.a_mn) off = (k / E) * (cs.M * 128) + sw128(m, (k % E) * elt);
    else off = (m / E) * (cs.K * 128) + sw128(k, (m % E) * elt);
    float v = A[i];
    if (cs.tf32) *(float*)(sA + off) = v;
    else *(__nv_bfloat16*)(sA + off) = __float2bfloat16_rn(v);
  }
  for (int i = threadIdx.x; i < cs.N * cs.K; i += blockDim.x) {
    int n = i / cs.K, k = i % cs.K;
    uint32_t off;
    if (!cs.b_mn) off = (k / E) * (cs.N * 128) + sw128(n, (k % E) * elt);
    else off = (n / E) * (cs.K * 128) + sw128(k, (n % E) * elt);
    float v = B[i];
    if (cs.tf32) *(float*)(sB + off) = v;
    else *(__nv_bfloat16*)(sB + off) = __float2bfloat16_rn(v);
  }
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) tmem_alloc<256>(&tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  if (threadIdx.x == 0) {
    const int KM = cs.tf32 ? 8 : 16;       // K per instruction
    uint32_t id = idesc(cs.tf32 ? FMT_TF32 : FMT_BF16, cs.tf32 ? FMT_TF32 : FMT_BF16, cs.M, cs.N, cs.a_mn, cs.b_mn);
    for (int k0 = 0; k0 < cs.K; k0 += KM) {
      uint64_t ad, bd;
      if (!cs.a_mn) ad = smem_desc_sw128(smem_u32(sA) + (k0 / E) * cs.M * 128 + (k0 % E) * elt, 16, 1024);
      else ad = smem_desc_sw128(smem_u32(sA) + k0 * 128, cs.K * 128, 1024);
      if (!cs.b_mn) bd = smem_desc_sw128(smem_u32(sB) + (k0 / E) * cs.N * 128 + (k0 % E) * elt, 16, 1024);
      else bd = smem_desc_sw128(smem_u32(sB) + k0 * 128, cs.K * 128, 1024);
      if (cs.tf32) mma_tf32(tmem, ad, bd, id, k0 > 0);
      else mma_bf16(tmem, ad, bd, id, k0 > 0);
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  // TMEM → global: thread t of warp w reads lane 32w + t (row), columns 16 at a time
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int row = warp * 32 + lane;
  for (int c0 = 0; c0 < cs.N; c0 += 16) {
    float v[16];
    tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
    if (row < cs.M)
      for (int j = 0; j < 16; ++j) D[row * cs.N + c0 + j] = v[j];
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<256>(tmem);
}

static float bf16r(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }
static float tf32_trunc(float x) { uint32_t u; memcpy(&u, &x, 4); u &= 0xFFFFE000u; float r; memcpy(&r, &u, 4); return r; }
static float h_tf32_rn(float x) {
  uint32_t u; memcpy(&u, &x, 4);
  u = (u + 0x1000u) & 0xFFFFE000u;   // round half away (cvt.rna)
  float r; memcpy(&r, &u, 4); return r;
}

static int run(const Case& cs, const char* name, int special) {
  std::vector<float> A(cs.M * cs.K), B(cs.N * cs.K), D(cs.M * cs.N);
  srand(1234);
  for (auto& v : A) v = special ? 1.0f + 3.0f * powf(2.f, -12.f) : (rand() / (float)RAND_MAX - 0.5f);
  for (auto& v : B) v = special ? 1.0f : (rand() / (float)RAND_MAX - 0.5f);
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaMemset(dD, 0, D.size() * 4);
  cudaFuncSetAttribute(tc_case_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  tc_case_kernel<<<1, 128, 140 * 1024>>>(cs, dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("%s: CUDA error %s\n", name, cudaGetErrorString(e)); return 1; }
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  double max_rn = 0, max_tr = 0, max_ex = 0, scale = 0;
  for (int m = 0; m < cs.M; ++m)
    for (int n = 0; n < cs.N; ++n) {
      double rn = 0, tr = 0, ex = 0;
      for (int k = 0; k < cs.K; ++k) {
        float a = A[m * cs.K + k], b = B[n * cs.K + k];
        ex += (double)a * b;
        if (cs.tf32) { rn += (double)h_tf32_rn(a) * h_tf32_rn(b); tr += (double)tf32_trunc(a) * tf32_trunc(b); }
        else { rn += (double)bf16r(a) * bf16r(b); tr = rn; }
      }
      double d = D[m * cs.N + n];
      max_rn = fmax(max_rn, fabs(d - rn)); max_tr = fmax(max_tr, fabs(d - tr)); max_ex = fmax(max_ex, fabs(d - ex));
      scale = fmax(scale, fabs(ex));
      if (special && m == 0 && n == 0) printf("  D[0][0]=%.9f exact=%.9f rn=%.9f trunc=%.9f\n", d, ex, rn, tr);
    }
  printf("%-34s max|D-ref_rn|=%.3e  max|D-ref_trunc|=%.3e  max|D-exact|=%.3e  (scale %.2f)\n", name, max_rn, max_tr,
         max_ex, scale);
  cudaFree(dA); cudaFree(dB); cudaFree(dD);
  return 0;
}

int main() {
  run({0, 0, 0, 128, 64, 64}, "bf16 A:K B:K M128 N64 K64", 0);
  run({0, 1, 0, 128, 64, 64}, "bf16 A:MN B:K M128 N64 K64", 0);
  run({0, 0, 1, 128, 64, 64}, "bf16 A:K B:MN M128 N64 K64", 0);
  run({0, 1, 1, 128, 128, 64}, "bf16 A:MN B:MN M128 N128 K64", 0);
  run({0, 0, 0, 128, 128, 128}, "bf16 A:K B:K M128 N128 K128", 0);
  run({1, 0, 0, 128, 64, 32}, "tf32 A:K B:K M128 N64 K32", 0);
  run({1, 1, 0, 128, 64, 32}, "tf32 A:MN B:K M128 N64 K32", 0);
  run({1, 0, 1, 128, 64, 32}, "tf32 A:K B:MN M128 N64 K32", 0);
  run({1, 0, 0, 128, 64, 32}, "tf32 rounding probe (1+3*2^-12)", 1);
  return 0;
}
