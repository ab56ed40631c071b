// Latency microbenchmarks for the one-CTA fp64 kernels (Cholesky / L⁻¹ / Ritz): what one "step" costs.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_small tools/microbench_small.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_sync(int iters, unsigned long long* out) {
  __shared__ double s[256];
  s[threadIdx.x] = threadIdx.x;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    s[threadIdx.x] += 1.0;
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
}

__global__ void k_rsqrt(int iters, double x, unsigned long long* out, double* sink) {
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = rsqrt(x) + 1.0;
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[1] = (t1 - t0) / iters; sink[0] = x; }
}

__global__ void k_sqrtdiv(int iters, double x, unsigned long long* out, double* sink) {
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = 1.0 / sqrt(x) + 1.0;
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[2] = (t1 - t0) / iters; sink[1] = x; }
}

__global__ void k_dfma(int iters, double x, unsigned long long* out, double* sink) {
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, 0.999, 0.001);
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[3] = (t1 - t0) / iters; sink[2] = x; }
}

__global__ void k_smem_chain(int iters, unsigned long long* out, double* sink) {
  __shared__ double s[512];
  for (int i = threadIdx.x; i < 512; i += blockDim.x) s[i] = i;
  __syncthreads();
  int idx = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    double v = s[idx];
    s[idx] = v * 0.5 + 1.0;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[4] = (t1 - t0) / iters; sink[3] = s[0]; }
}

// one Cholesky-like step: pivot read + rsqrt + 8 rows × 2 cols RMW + barrier
__global__ void k_step(int iters, unsigned long long* out, double* sink) {
  __shared__ double A[64 * 65];
  for (int i = threadIdx.x; i < 64 * 65; i += blockDim.x) A[i] = (i % 66 == 0) ? 100.0 : 0.01;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int j = it & 31;
    const double p = A[j * 65 + j];
    const double rp = rsqrt(p);
    const double r2 = rp * rp;
    for (int i = j + 1 + warp; i < 64; i += 8) {
      const double aij = A[i * 65 + j] * r2;
      for (int k = j + 1 + lane; k <= i; k += 32) A[i * 65 + k] -= aij * A[k * 65 + j] * 1e-9;
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[5] = (t1 - t0) / iters; sink[4] = A[5]; }
}

__global__ void k_step2(int iters, unsigned long long* out, double* sink) {
  __shared__ double A[64 * 65];
  for (int i = threadIdx.x; i < 64 * 65; i += blockDim.x) A[i] = (i % 66 == 0) ? 100.0 : 0.01;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = 8;
  const int m = 64, lda = 65;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int j = it & 31;
    const double p = A[j * lda + j];
    const double rp = rsqrt(p);
    const double r2 = rp * rp * 1e-9;
    double ck[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int k = j + 1 + lane + 32 * c;
      ck[c] = k < m ? A[k * lda + j] : 0.0;
    }
    for (int i0 = j + 1 + warp; i0 < m; i0 += 4 * nw) {
      double aij[4], v[4][4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u * nw;
        aij[u] = i < m ? A[i * lda + j] * r2 : 0.0;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int k = j + 1 + lane + 32 * c;
          v[u][c] = (i < m && k <= i) ? A[i * lda + k] : 0.0;
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u * nw;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int k = j + 1 + lane + 32 * c;
          if (i < m && k <= i) A[i * lda + k] = v[u][c] - aij[u] * ck[c];
        }
      }
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[6] = (t1 - t0) / iters; sink[5] = A[5]; }
}

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// one Householder tridiagonalisation sweep (m = 64) as in ritz_values_kernel; which = 0 full step,
// 1 without the matvec, 2 without the rank-2 update, 3 only barriers + reductions
__global__ void k_tridiag(int which, unsigned long long* out, double* sink) {
  extern __shared__ double A[];
  __shared__ double vec[128], pv[128];
  const int m = 64, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nt = blockDim.x, nw = nt >> 5;
  for (int i = tid; i < m * m; i += nt) A[i] = ((i / m) == (i % m) ? 2.0 : 0.0) + 1.0 / (1 + (i / m) + (i % m));
  __syncthreads();
  long long t0 = clock64();
  for (int k = 0; k + 2 < m; ++k) {
    const int n1 = m - k - 1;
    const double* col = A + (k + 1) * m + k;
    double ss = 0.0;
    for (int i = lane; i < n1; i += 32) ss += col[i * m] * col[i * m];
    ss = wsum(ss);
    const double x0 = col[0];
    const double alpha = ss > 0.0 ? -copysign(sqrt(ss), x0) : 0.0;
    const double v0 = x0 - alpha;
    const double vtv = ss - x0 * x0 + v0 * v0;
    const double beta = vtv > 0.0 ? 2.0 / vtv : 0.0;
    const double vi = tid < n1 ? (tid == 0 ? col[0] - alpha : col[tid * m]) : 0.0;
    __syncthreads();
    if (tid < n1) vec[tid] = vi;
    __syncthreads();
    if (which != 1 && which != 3) {
      for (int i = warp; i < n1; i += nw) {
        const double* row = A + (k + 1 + i) * m + (k + 1);
        double acc = 0.0;
        for (int j = lane; j < n1; j += 32) acc = fma(row[j], vec[j], acc);
        acc = wsum(acc);
        if (lane == 0) pv[i] = beta * acc;
      }
    }
    __syncthreads();
    double kk = 0.0;
    for (int i = lane; i < n1; i += 32) kk += vec[i] * pv[i];
    kk = wsum(kk);
    const double K = 0.5 * beta * kk;
    if (which != 2 && which != 3) {
      for (int i = warp; i < n1; i += nw) {
        const double vv = vec[i], ww = pv[i] - K * vv;
        double* Ai = A + (k + 1 + i) * m + (k + 1);
        for (int j = lane; j < n1; j += 32) Ai[j] -= vv * (pv[j] - K * vec[j]) + ww * vec[j];
      }
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) { out[7 + which] = (t1 - t0) / 62; sink[6] = A[7]; }
}

int main() {
  unsigned long long* out;
  double* sink;
  cudaMalloc(&out, 16 * sizeof(unsigned long long));
  cudaMalloc(&sink, 16 * sizeof(double));
  cudaMemset(out, 0, 16 * sizeof(unsigned long long));
  for (int rep = 0; rep < 2; ++rep) {
    k_sync<<<1, 256>>>(1000, out);
    k_rsqrt<<<1, 32>>>(1000, 2.0, out, sink);
    k_sqrtdiv<<<1, 32>>>(1000, 2.0, out, sink);
    k_dfma<<<1, 32>>>(1000, 2.0, out, sink);
    k_smem_chain<<<1, 256>>>(1000, out, sink);
    k_step<<<1, 256>>>(1000, out, sink);
    k_step2<<<1, 256>>>(1000, out, sink);
    for (int w = 0; w < 4; ++w) k_tridiag<<<1, 512, 64 * 64 * 8>>>(w, out, sink);
  }
  unsigned long long h[16];
  cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
  printf("cycles per iteration: syncthreads(256) %llu  rsqrt(f64) %llu  1/sqrt(f64) %llu  dfma %llu  smem RMW %llu  "
         "chol-step %llu  batched %llu\n", h[0], h[1], h[2], h[3], h[4], h[5], h[6]);
  printf("tridiag step cycles (512 thr): full %llu  no-matvec %llu  no-update %llu  sync+reductions %llu\n", h[7], h[8],
         h[9], h[10]);
  return 0;
}
