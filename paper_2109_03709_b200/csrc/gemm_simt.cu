// gemm_simt.cu — CUDA-core streaming products (see gemm_simt.cuh).
#include "gemm_simt.cuh"

namespace ppca {

// Load 8 consecutive elements of row r (k0..k0+7) as floats; zero outside [0,K).
template <typename T>
__device__ __forceinline__ void load8(const T* __restrict__ p, int64_t ld, int64_t r, int64_t R,
                                      int64_t k0, int64_t K, bool vec, float v[8]);

template <>
__device__ __forceinline__ void load8<float>(const float* __restrict__ p, int64_t ld, int64_t r,
                                             int64_t R, int64_t k0, int64_t K, bool vec, float v[8]) {
  if (r < R && vec && k0 + 8 <= K) {
    const float4* q = reinterpret_cast<const float4*>(p + r * ld + k0);
    float4 a = __ldg(q), b = __ldg(q + 1);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = (r < R && k0 + i < K) ? p[r * ld + k0 + i] : 0.f;
  }
}

template <>
__device__ __forceinline__ void load8<__nv_bfloat16>(const __nv_bfloat16* __restrict__ p, int64_t ld,
                                                     int64_t r, int64_t R, int64_t k0, int64_t K,
                                                     bool vec, float v[8]) {
  if (r < R && vec && k0 + 8 <= K) {
    uint4 u = __ldg(reinterpret_cast<const uint4*>(p + r * ld + k0));
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[2 * i] = __uint_as_float(w[i] << 16);
      v[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = (r < R && k0 + i < K) ? __bfloat162float(p[r * ld + k0 + i]) : 0.f;
  }
}

template <>
__device__ __forceinline__ void load8<SplitF32>(const SplitF32* __restrict__ p, int64_t ld, int64_t r, int64_t R,
                                                int64_t k0, int64_t K, bool vec, float v[8]) {
  // K = d (logical columns): the lo plane of the row starts K bf16 after the hi plane
  const __nv_bfloat16* row = reinterpret_cast<const __nv_bfloat16*>(p + (r < R ? r : 0) * ld);
  if (r < R && vec && k0 + 8 <= K) {
    uint4 h = __ldg(reinterpret_cast<const uint4*>(row + k0));
    uint4 l = __ldg(reinterpret_cast<const uint4*>(row + K + k0));
    const uint32_t wh[4] = {h.x, h.y, h.z, h.w}, wl[4] = {l.x, l.y, l.z, l.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[2 * i] = __uint_as_float(wh[i] << 16) + __uint_as_float(wl[i] << 16);
      v[2 * i + 1] = __uint_as_float(wh[i] & 0xffff0000u) + __uint_as_float(wl[i] & 0xffff0000u);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      v[i] = (r < R && k0 + i < K) ? __bfloat162float(row[k0 + i]) + __bfloat162float(row[K + k0 + i]) : 0.f;
  }
}

// ------------------------------------------------------------------------------------ NT
// Tile 128 (M) × 64 (N) × 16 (K); 256 threads, 8×4 outputs each.
constexpr int NT_BM = 128, NT_BN = 64, NT_BK = 16;

template <typename TX>
__global__ void __launch_bounds__(256) nt_kernel(const TX* __restrict__ A, int64_t lda,
                                                 const float* __restrict__ B, int64_t ldb,
                                                 float* __restrict__ C, int64_t ldc, int64_t M,
                                                 int64_t N, int64_t K, bool vecA, bool vecB) {
  __shared__ float As[NT_BK][NT_BM + 4];
  __shared__ float Bs[NT_BK][NT_BN + 4];
  const int tid = threadIdx.x;
  const int64_t m0 = (int64_t)blockIdx.x * NT_BM;
  const int64_t n0 = (int64_t)blockIdx.y * NT_BN;
  const int tx = tid % 16, ty = tid / 16;   // tx → N (4 each), ty → M (8 each)
  float acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  // loader mapping: A: row = tid/2 (0..127), k-half = tid%2;  B: row = tid/4 (0..63), k-quarter
  const int ar = tid >> 1, ak = (tid & 1) * 8;
  const int br = tid >> 2, bk = (tid & 3) * 4;
  for (int64_t k0 = 0; k0 < K; k0 += NT_BK) {
    float va[8];
    load8<TX>(A, lda, m0 + ar, M, k0 + ak, K, vecA, va);
#pragma unroll
    for (int i = 0; i < 8; ++i) As[ak + i][ar] = va[i];
    {
      int64_t r = n0 + br;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        int64_t k = k0 + bk + i;
        Bs[bk + i][br] = (r < N && k < K) ? __ldg(B + r * ldb + k) : 0.f;
      }
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < NT_BK; ++kk) {
      float a[8], b[4];
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = As[kk][ty * 8 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    int64_t r = m0 + ty * 8 + i;
    if (r >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int64_t cc = n0 + tx * 4 + j;
      if (cc < N) C[r * ldc + cc] = acc[i][j];
    }
  }
}

template <typename TX>
ppca_status launch_nt(Ctx* c, const TX* A, int64_t lda, const float* B, int64_t ldb, float* C,
                      int64_t ldc, int64_t M, int64_t N, int64_t K) {
  if (M <= 0 || N <= 0) return PPCA_OK;
  dim3 grid((unsigned)ceil_div(M, NT_BM), (unsigned)ceil_div(N, NT_BN));
  bool vecA = (lda * sizeof(TX)) % 16 == 0 && ((uintptr_t)A % 16) == 0;
  bool vecB = true;
  (void)vecB;
  nt_kernel<TX><<<grid, 256, 0, c->stream>>>(A, lda, B, ldb, C, ldc, M, N, K, vecA, true);
  PPCA_LAUNCH_CHECK(c, "nt_kernel");
  return PPCA_OK;
}

template ppca_status launch_nt<float>(Ctx*, const float*, int64_t, const float*, int64_t, float*,
                                      int64_t, int64_t, int64_t, int64_t);
template ppca_status launch_nt<__nv_bfloat16>(Ctx*, const __nv_bfloat16*, int64_t, const float*,
                                              int64_t, float*, int64_t, int64_t, int64_t, int64_t);
template ppca_status launch_nt<SplitF32>(Ctx*, const SplitF32*, int64_t, const float*, int64_t, float*, int64_t,
                                         int64_t, int64_t, int64_t);

// ------------------------------------------------------------------------------------ TN split-K
// Tile 64 (M) × 128 (N) × 16 (K rows); 256 threads, 4×8 outputs each; fp32 per slab → fp64.
constexpr int TN_BM = 64, TN_BN = 128, TN_BK = 16;

template <typename TA, typename TB>
__global__ void __launch_bounds__(256) tn_kernel(const TA* __restrict__ A, int64_t lda,
                                                 const TB* __restrict__ B, int64_t ldb,
                                                 double* __restrict__ P, int64_t M, int64_t N,
                                                 int64_t K, int64_t rows_per_split, bool vecA,
                                                 bool vecB) {
  __shared__ float As[TN_BK][TN_BM + 4];
  __shared__ float Bs[TN_BK][TN_BN + 4];
  const int tid = threadIdx.x;
  const int64_t m0 = (int64_t)blockIdx.y * TN_BM;      // M ≤ 128 (vectors): the y dimension
  const int64_t n0 = (int64_t)blockIdx.x * TN_BN;      // N = d can exceed 65535 tiles (huge d): x
  const int64_t kbeg = (int64_t)blockIdx.z * rows_per_split;
  const int64_t kend = min(K, kbeg + rows_per_split);
  const int tx = tid % 16, ty = tid / 16;    // tx → N (8 each), ty → M (4 each)
  double acc[4][8];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;
  // loaders: A slab 16 × 64: row = tid/16, cols (tid%16)*4..+4 ;  B slab 16 × 128: row = tid/16, cols (tid%16)*8..+8
  const int lr = tid >> 4, lc = tid & 15;
  for (int64_t k0 = kbeg; k0 < kend; k0 += TN_BK) {
    {
      float va[8];
      // A is [K][M]: row k0+lr, columns m0 + lc*4 .. +4 (use load8 on the first 4 only)
      int64_t r = k0 + lr;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        int64_t col = m0 + lc * 4 + i;
        va[i] = (r < kend && col < M) ? load_rc(A, lda, r, col, M) : 0.f;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) As[lr][lc * 4 + i] = va[i];
    }
    {
      float vb[8];
      int64_t r = k0 + lr;
      load8<TB>(B, ldb, r, kend, n0 + lc * 8, N, vecB, vb);
#pragma unroll
      for (int i = 0; i < 8; ++i) Bs[lr][lc * 8 + i] = vb[i];
    }
    __syncthreads();
    float part[4][8];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) part[i][j] = 0.f;
#pragma unroll
    for (int kk = 0; kk < TN_BK; ++kk) {
      float a[4], b[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 8; ++j) b[j] = Bs[kk][tx * 8 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) part[i][j] = fmaf(a[i], b[j], part[i][j]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j] += (double)part[i][j];
    __syncthreads();
  }
  double* Pz = P + (int64_t)blockIdx.z * M * N;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int64_t r = m0 + ty * 4 + i;
    if (r >= M) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      int64_t cc = n0 + tx * 8 + j;
      if (cc < N) Pz[r * N + cc] = acc[i][j];
    }
  }
}

int tn_pick_splits(Ctx* c, int64_t M, int64_t N, int64_t K) {
  int64_t tiles = ceil_div(M, TN_BM) * ceil_div(N, TN_BN);
  int64_t want = ceil_div(4 * (int64_t)c->sm_count, tiles);
  int64_t maxs = ceil_div(K, 4 * TN_BK);           // at least 64 rows per split
  int64_t s = want < maxs ? want : maxs;
  if (s < 1) s = 1;
  if (s > 1024) s = 1024;
  return (int)s;
}

template <typename TA, typename TB>
ppca_status launch_tn_splitk(Ctx* c, const TA* A, int64_t lda, const TB* B, int64_t ldb,
                             double* P, int64_t M, int64_t N, int64_t K, int nsplit) {
  if (M <= 0 || N <= 0) return PPCA_OK;
  int64_t rps = ceil_div(ceil_div(K > 0 ? K : 1, nsplit), TN_BK) * TN_BK;
  if (ceil_div(M, TN_BM) > 65535) return set_error(c, PPCA_ERR_UNSUPPORTED, "tn_kernel: M = %lld", (long long)M);
  dim3 grid((unsigned)ceil_div(N, TN_BN), (unsigned)ceil_div(M, TN_BM), (unsigned)nsplit);
  bool vecB = (ldb * sizeof(TB)) % 16 == 0 && ((uintptr_t)B % 16) == 0;
  tn_kernel<TA, TB><<<grid, 256, 0, c->stream>>>(A, lda, B, ldb, P, M, N, K, rps, false, vecB);
  PPCA_LAUNCH_CHECK(c, "tn_kernel");
  return PPCA_OK;
}

template ppca_status launch_tn_splitk<float, float>(Ctx*, const float*, int64_t, const float*, int64_t,
                                                    double*, int64_t, int64_t, int64_t, int);
template ppca_status launch_tn_splitk<__nv_bfloat16, __nv_bfloat16>(Ctx*, const __nv_bfloat16*, int64_t,
                                                                    const __nv_bfloat16*, int64_t, double*,
                                                                    int64_t, int64_t, int64_t, int);
template ppca_status launch_tn_splitk<float, __nv_bfloat16>(Ctx*, const float*, int64_t,
                                                            const __nv_bfloat16*, int64_t, double*,
                                                            int64_t, int64_t, int64_t, int);
template ppca_status launch_tn_splitk<SplitF32, SplitF32>(Ctx*, const SplitF32*, int64_t, const SplitF32*, int64_t,
                                                          double*, int64_t, int64_t, int64_t, int);
template ppca_status launch_tn_splitk<float, SplitF32>(Ctx*, const float*, int64_t, const SplitF32*, int64_t,
                                                       double*, int64_t, int64_t, int64_t, int);

// ------------------------------------------------------------------------------------ reductions
__global__ void reduce_splits_f32_kernel(const double* __restrict__ P, int nsplit, int64_t count,
                                         float* __restrict__ out, int64_t ldo, int64_t cols) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  double s = 0.0;
  for (int z = 0; z < nsplit; ++z) s += P[(int64_t)z * count + i];
  int64_t r = i / cols, cc = i % cols;
  out[r * ldo + cc] = (float)s;
}

// out[i] = Σ_z P[z][i]: block = 32 outputs (lanes, coalesced) × 8 warps; warp w sums the splits z ≡ w (mod 8)
// with 8 loads in flight, the 8 warp sums are added in warp order (fixed order: deterministic).  A thread per
// output summing every split waited nsplit/8 dependent round trips (128 splits: 14 µs).
__global__ void __launch_bounds__(256) reduce_splits_f64_kernel(const double* __restrict__ P, int nsplit, int64_t count,
                                                                double* __restrict__ out) {
  pdl_enter();
  __shared__ double part[8][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t i = (int64_t)blockIdx.x * 32 + lane;
  double s = 0.0;
  if (i < count) s = sum_in_order<8>(warp, nsplit, 8, [&](int64_t z) { return P[z * count + i]; });
  part[warp][lane] = s;
  __syncthreads();
  if (warp == 0 && i < count) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += part[w][lane];
    out[i] = t;
  }
}

ppca_status launch_reduce_splits_f32(Ctx* c, const double* P, int nsplit, int64_t count, float* out,
                                     int64_t ldo, int64_t cols) {
  if (count <= 0) return PPCA_OK;
  reduce_splits_f32_kernel<<<(unsigned)ceil_div(count, 256), 256, 0, c->stream>>>(P, nsplit, count, out,
                                                                                  ldo, cols);
  PPCA_LAUNCH_CHECK(c, "reduce_splits_f32");
  return PPCA_OK;
}

ppca_status launch_reduce_splits_f64(Ctx* c, const double* P, int nsplit, int64_t count, double* out) {
  return launch_reduce_splits_f64(c, P, nsplit, count, out, c->stream);
}

ppca_status launch_reduce_splits_f64(Ctx* c, const double* P, int nsplit, int64_t count, double* out,
                                     cudaStream_t st) {
  if (count <= 0) return PPCA_OK;
  launch_pdl(reduce_splits_f64_kernel, dim3((unsigned)ceil_div(count, (int64_t)32)), dim3(256), 0, st, P, nsplit, count, out);
  PPCA_LAUNCH_CHECK(c, "reduce_splits_f64");
  return PPCA_OK;
}

}  // namespace ppca
