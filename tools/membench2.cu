// membench2.cu — converter-like streaming read (LDG.128 → registers → STS) on B200: how many warps and
// register buffers does one CTA per SM need to approach HBM bandwidth?  Random data (no compression).
#include <cstdio>
#include <cuda_runtime.h>

template <int NBUF>
__global__ void conv(const float* __restrict__ X, long n, long d, float* out) {
  extern __shared__ __align__(16) float4 buf[];          // [NBUF][8][blockDim]
  const int nw = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sub = lane >> 4, cl = lane & 15;
  const int rpw = 128 / nw;                              // rows per warp per chunk
  const int ipw = rpw / 2;                               // loads per thread per chunk
  const long ntiles = (n + 127) / 128, nk = d / 64;
  const long nch = ((ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x) * nk;
  float4 R[NBUF][8];
  long lt = blockIdx.x, lk = 0;
  auto load = [&](float4 (&r)[8]) {
    const long row0 = lt * 128 + warp * rpw + sub;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float4 v = make_float4(0, 0, 0, 0);
      if (i < ipw && row0 + 2 * i < n) v = __ldcs(reinterpret_cast<const float4*>(X + (row0 + 2 * i) * d + lk * 64 + cl * 4));
      r[i] = v;
    }
    if (++lk == nk) { lk = 0; lt += gridDim.x; }
  };
  auto store = [&](int slot, const float4 (&r)[8]) {
#pragma unroll
    for (int i = 0; i < 8; ++i) if (i < ipw) buf[(slot * 8 + i) * blockDim.x + threadIdx.x] = r[i];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
  };
#pragma unroll
  for (int b = 0; b < NBUF - 1; ++b) load(R[b]);
  for (long c = 0; c < nch; c += NBUF) {
#pragma unroll
    for (int b = 0; b < NBUF; ++b) {
      if (c + b >= nch) break;
      load(R[(b + NBUF - 1) % NBUF]);
      store(b, R[b]);
    }
  }
  __syncthreads();
  float s = 0;
  for (int i = threadIdx.x; i < NBUF * 8 * (int)blockDim.x; i += blockDim.x) s += buf[i].x;
  if (s == 1234.5f) out[0] = 1.f;
}

__global__ void fill(float* X, long count) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < count; i += (long)gridDim.x * blockDim.x) {
    unsigned h = (unsigned)(i * 2654435761u) ^ (unsigned)(i >> 7) * 40503u;
    X[i] = (float)(h & 0xffffff) * 1e-7f - 0.8f;
  }
}

template <int NB>
void run(const float* X, long n, long d, float* out, int threads) {
  size_t smem = (size_t)NB * 8 * threads * 16;
  cudaFuncSetAttribute(conv<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    conv<NB><<<148, threads, smem>>>(X, n, d, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (rep == 2) printf("warps=%2d buffers=%d (loads/thread/chunk %d): %.3f ms  %.0f GB/s  err=%s\n", threads / 32, NB,
                         128 / (threads / 32) / 2, ms, n * d * 4.0 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  }
}

int main() {
  long n = 1000000, d = 1024;
  float* X; float* out;
  cudaMalloc(&X, n * d * 4); cudaMalloc(&out, 4);
  fill<<<4096, 256>>>(X, n * d);
  run<2>(X, n, d, out, 256);
  run<3>(X, n, d, out, 256);
  run<4>(X, n, d, out, 256);
  run<2>(X, n, d, out, 512);
  run<3>(X, n, d, out, 512);
  run<2>(X, n, d, out, 1024);
  return 0;
}
