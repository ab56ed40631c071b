// membench.cu — how the row-run length of a tiled fp32 read affects HBM throughput on B200.
// Reads an n × d fp32 matrix in tiles of R rows × C columns (C contiguous floats per row), tile-major
// with the column chunks of a row tile consecutive (the order a K-loop reads them), 148 persistent CTAs.
#include <cstdio>
#include <cuda_runtime.h>

template <int C, int NBUF>
__global__ void __launch_bounds__(256) rd(const float* __restrict__ X, long n, long d, int R, float* out) {
  // 8 warps; lanes cover C/4 float4 of a row; rows per warp instruction = 32 / (C/4)
  constexpr int LPR = C / 4;                  // lanes per row
  constexpr int RPI = 32 / LPR;               // rows per instruction
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sub = lane / LPR, cl = lane % LPR;
  float acc = 0.f;
  const long ntiles = (n + R - 1) / R, nk = d / C;
  const int ipw = R / (8 * RPI);               // instructions per warp per chunk
  for (long t = blockIdx.x; t < ntiles; t += gridDim.x)
    for (long kc = 0; kc < nk; ++kc) {
      float4 v[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        if (i < ipw) {
          long row = t * R + (warp * ipw + i) * RPI + sub;
          v[i] = row < n ? __ldcs(reinterpret_cast<const float4*>(X + row * d + kc * C + cl * 4)) : make_float4(0, 0, 0, 0);
        }
      }
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (i < ipw) acc += v[i].x + v[i].y + v[i].z + v[i].w;
    }
  if (acc == 1234.5f) out[0] = acc;
}

template <int C>
void run(const float* X, long n, long d, int R, float* out) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    rd<C, 1><<<148 * 2, 256>>>(X, n, d, R, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (rep == 2) printf("R=%4d C=%4d (row run %5d B): %.3f ms  %.0f GB/s\n", R, C, C * 4, ms, n * d * 4.0 / ms / 1e6);
  }
}

int main() {
  long n = 1000000, d = 1024;
  float* X; float* out;
  cudaMalloc(&X, n * d * 4); cudaMalloc(&out, 4);
  cudaMemset(X, 0x3f, n * d * 4);
  run<64>(X, n, d, 128, out);    // kernel A pattern: 256 B runs
  run<64>(X, n, d, 256, out);
  run<128>(X, n, d, 128, out);   // 512 B runs
  run<128>(X, n, d, 64, out);

  return 0;
}
