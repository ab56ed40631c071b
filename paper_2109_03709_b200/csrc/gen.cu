// gen.cu — ppca_generate: the seeded synthetic workloads on the device (support row a8).
//
// Same recipe as inputs/generate.py, implemented independently:
//   planted_qr:          x = Q(√λ∘g), Q = Q-factor (positive diag R) of Γ, by modified Gram–Schmidt
//                        on the device in fp64;  μ = Q(√λ∘ḡ) (linearity; ḡ = column means of g)
//   planted_householder: x = relu(H_1⋯H_r(√λ∘g)); the r reflection coefficients of each row are
//                        obtained from the r dot products u_i·y and the r×r Gram of the u_i
//   image_factor:        x = mask∘clip((0.13/50)·a·B, 0, 1)
// All raw values are fp64; X = RNE_storage(raw − μ).  Column means are fp64 over all n rows
// (per-rank partial sums + all-reduce).
#include "common.cuh"
#include "gemm_simt.cuh"

namespace ppca {

struct RowMap {
  int layout;          // 0 contiguous, 1 interleaved
  int64_t n, b, row0;  // row0: first global row (contiguous)
  int rank, world;
  __host__ __device__ int64_t operator()(int64_t li) const {
    if (layout == 0) return row0 + li;
    int64_t q = b / world;
    int64_t nbf = n / b;
    if (li < nbf * q) return (li / q) * b + rank * q + (li % q);
    int64_t p = n - nbf * b;
    int64_t qt = p / world;
    return nbf * b + rank * qt + (li - nbf * q);
  }
};

__device__ __forceinline__ double lambda_j(int spectrum, double a, double noise, int64_t j /*0-based*/) {
  double jj = (double)(j + 1);
  return (spectrum == PPCA_SPECTRUM_EXP ? exp(-jj / a) : pow(jj, -a)) + noise;
}

template <typename T>
__device__ __forceinline__ void store_val(T* p, double v);
template <>
__device__ __forceinline__ void store_val<float>(float* p, double v) { *p = (float)v; }
template <>
__device__ __forceinline__ void store_val<__nv_bfloat16>(__nv_bfloat16* p, double v) { *p = f64_to_bf16_rne(v); }

// ----------------------------------------------------------------------------- planted QR
// QT[j][i] = Γ[i][j]  (row j of QT = column j of Γ)
__global__ void gamma_kernel(uint64_t seed, int64_t d, double* __restrict__ QT) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= d * d) return;
  int64_t j = e / d, i = e % d;
  QT[e] = gaussian_elt(seed, 1u, (uint64_t)(i * d + j));
}

// right-looking MGS step j: for rows i > j:  a_i ← a_i − (a_j·a_i / a_j·a_j) a_j
__global__ void mgs_step_kernel(double* __restrict__ QT, int64_t d, int64_t j) {
  int64_t i = j + 1 + blockIdx.x;
  const double* aj = QT + j * d;
  double* ai = QT + i * d;
  double nn = 0.0, dt = 0.0;
  for (int64_t x = threadIdx.x; x < d; x += blockDim.x) {
    double v = aj[x];
    nn += v * v;
    dt += v * ai[x];
  }
  nn = warp_sum(nn);
  dt = warp_sum(dt);
  __shared__ double r0[32], r1[32];
  __shared__ double coef;
  if ((threadIdx.x & 31) == 0) { r0[threadIdx.x >> 5] = nn; r1[threadIdx.x >> 5] = dt; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0, b = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { a += r0[w]; b += r1[w]; }
    coef = b / a;
  }
  __syncthreads();
  for (int64_t x = threadIdx.x; x < d; x += blockDim.x) ai[x] -= coef * aj[x];
}

// rows normalised, then scaled by √λ_j:  B[j][i] = √λ_j · q_j[i]
__global__ void qt_finish_kernel(double* __restrict__ QT, int64_t d, int spectrum, double a, double noise) {
  int64_t j = blockIdx.x;
  double* q = QT + j * d;
  double nn = 0.0;
  for (int64_t x = threadIdx.x; x < d; x += blockDim.x) nn += q[x] * q[x];
  nn = warp_sum(nn);
  __shared__ double r0[32];
  __shared__ double sc;
  if ((threadIdx.x & 31) == 0) r0[threadIdx.x >> 5] = nn;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += r0[w];
    sc = sqrt(lambda_j(spectrum, a, noise, j)) / sqrt(t);
  }
  __syncthreads();
  for (int64_t x = threadIdx.x; x < d; x += blockDim.x) q[x] *= sc;
}

// column sums of g over this rank's rows (fp64 partials [split][d])
__global__ void colsum_gauss_kernel(uint64_t seed, RowMap rm, int64_t n_local, int64_t d,
                                    int64_t rows_per_split, double* __restrict__ P) {
  int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= d) return;
  int64_t r0 = (int64_t)blockIdx.y * rows_per_split, r1 = min(n_local, r0 + rows_per_split);
  double s = 0.0;
  for (int64_t li = r0; li < r1; ++li) s += gaussian_elt(seed, 0u, (uint64_t)(rm(li) * d + j));
  P[(int64_t)blockIdx.y * d + j] = s;
}

// μ_i = Σ_j B[j][i] gsum_j / n
__global__ void planted_mean_kernel(const double* __restrict__ B, const double* __restrict__ gsum, int64_t d,
                                    double inv_n, double* __restrict__ mu) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= d) return;
  double s = 0.0;
  for (int64_t j = 0; j < d; ++j) s += B[j * d + i] * gsum[j];
  mu[i] = s * inv_n;
}

// panel of g rows (fp64), local rows [l0, l0+rows)
__global__ void gauss_panel_kernel(uint64_t seed, RowMap rm, int64_t l0, int64_t rows, int64_t d,
                                   double* __restrict__ Gp) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * d) return;
  int64_t r = e / d, j = e % d;
  Gp[e] = gaussian_elt(seed, 0u, (uint64_t)(rm(l0 + r) * d + j));
}

// X[l0+r][i] = RN( Σ_j Gp[r][j] B[j][i] − μ_i ); fp64 SIMT GEMM, tile 64×64×16, 4×4 per thread.
template <typename T>
__global__ void __launch_bounds__(256) planted_gemm_kernel(const double* __restrict__ Gp, const double* __restrict__ B,
                                                           const double* __restrict__ mu, int64_t rows, int64_t d,
                                                           T* __restrict__ X, int64_t ld) {
  __shared__ double As[16][65];
  __shared__ double Bs[16][65];
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  const int64_t r0 = (int64_t)blockIdx.y * 64, c0 = (int64_t)blockIdx.x * 64;
  double acc[4][4] = {};
  for (int64_t k0 = 0; k0 < d; k0 += 16) {
    for (int e = tid; e < 64 * 16; e += 256) {
      int rr = e / 16, kk = e % 16;
      int64_t r = r0 + rr, k = k0 + kk;
      As[kk][rr] = (r < rows && k < d) ? Gp[r * d + k] : 0.0;
      int kb = e / 64, cb = e % 64;
      int64_t kq = k0 + kb, cq = c0 + cb;
      Bs[kb][cb] = (kq < d && cq < d) ? B[kq * d + cq] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int64_t r = r0 + ty * 4 + i;
    if (r >= rows) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int64_t cc = c0 + tx * 4 + j;
      if (cc < d) store_val<T>(X + r * ld + cc, acc[i][j] - mu[cc]);
    }
  }
}

// ----------------------------------------------------------------------------- Householder
__global__ void house_u_kernel(uint64_t seed, int r, int64_t d, double* __restrict__ U) {
  int i = blockIdx.x;
  double nn = 0.0;
  for (int64_t x = threadIdx.x; x < d; x += blockDim.x) {
    double v = gaussian_elt(seed, 2u, (uint64_t)(i * d + x));
    U[i * d + x] = v;
    nn += v * v;
  }
  nn = warp_sum(nn);
  __shared__ double r0[32];
  __shared__ double inv;
  if ((threadIdx.x & 31) == 0) r0[threadIdx.x >> 5] = nn;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += r0[w];
    inv = 1.0 / sqrt(t);
  }
  __syncthreads();
  for (int64_t x = threadIdx.x; x < d; x += blockDim.x) U[i * d + x] *= inv;
}

constexpr int HMAX = 16;

__global__ void sqrt_lambda_kernel(int64_t d, int spectrum, double a, double noise, double* __restrict__ sl) {
  int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < d) sl[j] = sqrt(lambda_j(spectrum, a, noise, j));
}

// Mg[i][j] = u_i·u_j (one block per pair)
__global__ void house_gram_kernel(const double* __restrict__ U, int r, int64_t d, double* __restrict__ Mg) {
  int i = blockIdx.x / r, j = blockIdx.x % r;
  double s = 0.0;
  for (int64_t x = threadIdx.x; x < d; x += blockDim.x) s += U[i * d + x] * U[j * d + x];
  s = warp_sum(s);
  __shared__ double r0[32];
  if ((threadIdx.x & 31) == 0) r0[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += r0[w];
    Mg[i * r + j] = t;
  }
}

// per row: p_i = u_i·y (y = √λ∘g), c_i = p_i − 2 Σ_{j>i} c_j (u_i·u_j)   (H_{r-1} applied first)
__global__ void house_coef_kernel(uint64_t seed, RowMap rm, int64_t d, int r, const double* __restrict__ U,
                                  const double* __restrict__ sl, const double* __restrict__ Mg,
                                  double* __restrict__ coef) {
  int64_t li = blockIdx.x;
  int64_t gr = rm(li);
  double p[HMAX];
  for (int i = 0; i < r; ++i) p[i] = 0.0;
  for (int64_t x = threadIdx.x; x < d; x += blockDim.x) {
    double y = gaussian_elt(seed, 0u, (uint64_t)(gr * d + x)) * sl[x];
    for (int i = 0; i < r; ++i) p[i] += U[i * d + x] * y;
  }
  __shared__ double red[HMAX][32];
  for (int i = 0; i < r; ++i) {
    double v = warp_sum(p[i]);
    if ((threadIdx.x & 31) == 0) red[i][threadIdx.x >> 5] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double pp[HMAX], cc[HMAX];
    for (int i = 0; i < r; ++i) {
      double t = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[i][w];
      pp[i] = t;
    }
    for (int i = r - 1; i >= 0; --i) {
      double s = pp[i];
      for (int j = i + 1; j < r; ++j) s -= 2.0 * cc[j] * Mg[i * r + j];
      cc[i] = s;
    }
    for (int i = 0; i < r; ++i) coef[li * HMAX + i] = cc[i];
  }
}

__device__ __forceinline__ double house_val(uint64_t seed, int64_t gr, int64_t d, int64_t x, int r,
                                            const double* U, const double* cf, const double* sl, int relu) {
  double v = gaussian_elt(seed, 0u, (uint64_t)(gr * d + x)) * sl[x];
  for (int i = 0; i < r; ++i) v -= 2.0 * cf[i] * U[i * d + x];
  return relu ? fmax(v, 0.0) : v;
}

// ----------------------------------------------------------------------------- image factor
__global__ void image_a_kernel(uint64_t seed, RowMap rm, int64_t n_local, int rank_k, double* __restrict__ A) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n_local * rank_k) return;
  int64_t li = e / rank_k, t = e % rank_k;
  A[e] = exponential_elt(seed, 3u, (uint64_t)(rm(li) * rank_k + t));
}
__global__ void image_b_kernel(uint64_t seed, int rank_k, int64_t d, double* __restrict__ B) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rank_k * d) return;
  B[e] = exponential_elt(seed, 4u, (uint64_t)e);
}
__device__ __forceinline__ double image_val(uint64_t seed, int64_t gr, int64_t li, int64_t d, int64_t x,
                                            int rank_k, const double* A, const double* B) {
  double s = 0.0;
  for (int t = 0; t < rank_k; ++t) s += A[li * rank_k + t] * B[t * d + x];
  s = fmin(fmax(s * (0.13 / rank_k), 0.0), 1.0);
  double u = u32_to_unit(philox_word(seed, 5u, (uint64_t)(gr * d + x)));
  return u < 0.8 ? 0.0 : s;
}

// ----------------------------------------------------------------------------- generic colsum / store
struct GenArgs {
  int family, spectrum, relu, r, rank_k;
  double a, noise;
  uint64_t seed;
  int64_t d;
  const double* U;     // householder vectors
  const double* sl;    // √λ
  const double* coef;  // householder per-row coefficients [n_local][HMAX]
  const double* A;     // image A [n_local][rank]
  const double* B;     // image B [rank][d]
};

__device__ __forceinline__ double raw_val(const GenArgs& g, RowMap rm, int64_t li, int64_t x) {
  int64_t gr = rm(li);
  if (g.family == PPCA_PLANTED_HOUSEHOLDER)
    return house_val(g.seed, gr, g.d, x, g.r, g.U, g.coef + li * HMAX, g.sl, g.relu);
  return image_val(g.seed, gr, li, g.d, x, g.rank_k, g.A, g.B);
}

__global__ void colsum_raw_kernel(GenArgs g, RowMap rm, int64_t n_local, int64_t rows_per_split,
                                  double* __restrict__ P) {
  int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= g.d) return;
  int64_t r0 = (int64_t)blockIdx.y * rows_per_split, r1 = min(n_local, r0 + rows_per_split);
  double s = 0.0;
  for (int64_t li = r0; li < r1; ++li) s += raw_val(g, rm, li, j);
  P[(int64_t)blockIdx.y * g.d + j] = s;
}

template <typename T>
__global__ void store_raw_kernel(GenArgs g, RowMap rm, int64_t n_local, const double* __restrict__ mu,
                                 T* __restrict__ X, int64_t ld) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n_local * g.d) return;
  int64_t li = e / g.d, x = e % g.d;
  store_val<T>(X + li * ld + x, raw_val(g, rm, li, x) - mu[x]);
}

__global__ void scale_kernel(double* v, int64_t n, double s) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] *= s;
}

// ----------------------------------------------------------------------------- driver
static int64_t local_rows(const ppca_gen_spec* s, int rank, int world, int64_t* row0) {
  if (s->layout == PPCA_LAYOUT_CONTIGUOUS) {
    int64_t per = ceil_div(s->n_global, world);
    int64_t a = std::min(s->n_global, per * rank), b = std::min(s->n_global, per * (rank + 1));
    *row0 = a;
    return b - a;
  }
  int64_t b = s->block_rows, n = s->n_global;
  int64_t nbf = n / b, p = n - nbf * b;
  *row0 = 0;
  return nbf * (b / world) + p / world;
}

template <typename T>
static ppca_status generate_t(Ctx* c, const ppca_gen_spec* s, T* X, int64_t ld, int64_t n_local, RowMap rm,
                              double* mu) {
  const int64_t d = s->d;
  const int64_t n = s->n_global;
  int nsplit = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n_local, 256), 512));
  int64_t rps = std::max<int64_t>(1, ceil_div(n_local, nsplit));
  double* P = (double*)scratch(c, S_PART, (size_t)nsplit * d * sizeof(double));
  if (!P) return set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
  if (s->family == PPCA_PLANTED_QR) {
    double* QT = (double*)scratch(c, S_GEN0, (size_t)d * d * sizeof(double));
    if (!QT) return set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
    gamma_kernel<<<(unsigned)ceil_div(d * d, 256), 256, 0, c->stream>>>(s->seed, d, QT);
    PPCA_LAUNCH_CHECK(c, "gamma");
    for (int64_t j = 0; j + 1 < d; ++j) {
      mgs_step_kernel<<<(unsigned)(d - j - 1), 128, 0, c->stream>>>(QT, d, j);
      PPCA_LAUNCH_CHECK(c, "mgs_step");
    }
    qt_finish_kernel<<<(unsigned)d, 128, 0, c->stream>>>(QT, d, s->spectrum, s->a, s->noise);
    PPCA_LAUNCH_CHECK(c, "qt_finish");
    // mean
    if (n_local > 0) {
      colsum_gauss_kernel<<<dim3((unsigned)ceil_div(d, 128), nsplit), 128, 0, c->stream>>>(s->seed, rm, n_local, d,
                                                                                          rps, P);
      PPCA_LAUNCH_CHECK(c, "colsum_gauss");
      PPCA_TRY(launch_reduce_splits_f64(c, P, nsplit, d, mu));
    } else {
      PPCA_TRY(check_cuda(c, cudaMemsetAsync(mu, 0, d * sizeof(double), c->stream), "memset"));
    }
    PPCA_TRY(allreduce(c, mu, d, true));
    double* gs = (double*)scratch(c, S_GEN2, (size_t)d * sizeof(double));
    PPCA_TRY(check_cuda(c, cudaMemcpyAsync(gs, mu, d * sizeof(double), cudaMemcpyDeviceToDevice, c->stream), "cp"));
    planted_mean_kernel<<<(unsigned)ceil_div(d, 128), 128, 0, c->stream>>>(QT, gs, d, 1.0 / (double)n, mu);
    PPCA_LAUNCH_CHECK(c, "planted_mean");
    // panels
    int64_t panel = std::max<int64_t>(64, std::min<int64_t>(n_local, (int64_t)(256ll << 20) / (8 * d)));
    panel = (panel / 64) * 64;
    if (panel < 64) panel = 64;
    double* Gp = (double*)scratch(c, S_GEN1, (size_t)panel * d * sizeof(double));
    if (!Gp) return set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
    for (int64_t l0 = 0; l0 < n_local; l0 += panel) {
      int64_t rows = std::min(panel, n_local - l0);
      gauss_panel_kernel<<<(unsigned)ceil_div(rows * d, 256), 256, 0, c->stream>>>(s->seed, rm, l0, rows, d, Gp);
      PPCA_LAUNCH_CHECK(c, "gauss_panel");
      planted_gemm_kernel<T><<<dim3((unsigned)ceil_div(d, 64), (unsigned)ceil_div(rows, 64)), 256, 0, c->stream>>>(
          Gp, QT, mu, rows, d, X + l0 * ld, ld);
      PPCA_LAUNCH_CHECK(c, "planted_gemm");
    }
    return PPCA_OK;
  }
  GenArgs g{};
  g.family = s->family; g.spectrum = s->spectrum; g.relu = s->relu; g.r = s->house_r; g.rank_k = s->rank;
  g.a = s->a; g.noise = s->noise; g.seed = s->seed; g.d = d;
  if (s->family == PPCA_PLANTED_HOUSEHOLDER) {
    if (s->house_r < 1 || s->house_r > HMAX) return set_error(c, PPCA_ERR_INVALID_ARG, "house_r must be 1..%d", HMAX);
    double* U = (double*)scratch(c, S_GEN0, (size_t)s->house_r * d * sizeof(double));
    double* cf = (double*)scratch(c, S_GEN1, (size_t)std::max<int64_t>(1, n_local) * HMAX * sizeof(double));
    double* sl = (double*)scratch(c, S_GEN2, (size_t)(d + HMAX * HMAX) * sizeof(double));
    if (!U || !cf || !sl) return set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
    double* Mg = sl + d;
    sqrt_lambda_kernel<<<(unsigned)ceil_div(d, 256), 256, 0, c->stream>>>(d, s->spectrum, s->a, s->noise, sl);
    PPCA_LAUNCH_CHECK(c, "sqrt_lambda");
    house_u_kernel<<<s->house_r, 256, 0, c->stream>>>(s->seed, s->house_r, d, U);
    PPCA_LAUNCH_CHECK(c, "house_u");
    house_gram_kernel<<<s->house_r * s->house_r, 256, 0, c->stream>>>(U, s->house_r, d, Mg);
    PPCA_LAUNCH_CHECK(c, "house_gram");
    if (n_local > 0) {
      house_coef_kernel<<<(unsigned)n_local, 256, 0, c->stream>>>(s->seed, rm, d, s->house_r, U, sl, Mg, cf);
      PPCA_LAUNCH_CHECK(c, "house_coef");
    }
    g.U = U; g.coef = cf; g.sl = sl;
  } else if (s->family == PPCA_IMAGE_FACTOR) {
    if (s->rank < 1) return set_error(c, PPCA_ERR_INVALID_ARG, "rank must be >= 1");
    double* A = (double*)scratch(c, S_GEN0, (size_t)std::max<int64_t>(1, n_local) * s->rank * sizeof(double));
    double* B = (double*)scratch(c, S_GEN1, (size_t)s->rank * d * sizeof(double));
    if (!A || !B) return set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
    if (n_local > 0) {
      image_a_kernel<<<(unsigned)ceil_div(n_local * s->rank, 256), 256, 0, c->stream>>>(s->seed, rm, n_local,
                                                                                        s->rank, A);
      PPCA_LAUNCH_CHECK(c, "image_a");
    }
    image_b_kernel<<<(unsigned)ceil_div((int64_t)s->rank * d, 256), 256, 0, c->stream>>>(s->seed, s->rank, d, B);
    PPCA_LAUNCH_CHECK(c, "image_b");
    g.A = A; g.B = B;
  } else {
    return set_error(c, PPCA_ERR_INVALID_ARG, "unknown family %d", (int)s->family);
  }
  if (n_local > 0) {
    colsum_raw_kernel<<<dim3((unsigned)ceil_div(d, 128), nsplit), 128, 0, c->stream>>>(g, rm, n_local, rps, P);
    PPCA_LAUNCH_CHECK(c, "colsum_raw");
    PPCA_TRY(launch_reduce_splits_f64(c, P, nsplit, d, mu));
  } else {
    PPCA_TRY(check_cuda(c, cudaMemsetAsync(mu, 0, d * sizeof(double), c->stream), "memset"));
  }
  PPCA_TRY(allreduce(c, mu, d, true));
  scale_kernel<<<(unsigned)ceil_div(d, 256), 256, 0, c->stream>>>(mu, d, 1.0 / (double)n);
  PPCA_LAUNCH_CHECK(c, "scale");
  if (n_local > 0) {
    store_raw_kernel<T><<<(unsigned)ceil_div(n_local * d, 256), 256, 0, c->stream>>>(g, rm, n_local, mu, X, ld);
    PPCA_LAUNCH_CHECK(c, "store_raw");
  }
  return PPCA_OK;
}

ppca_status split_f32(Ctx* c, void* X, int64_t n_local, int64_t d, int64_t ld);

ppca_status generate(Ctx* c, const ppca_gen_spec* s, void* X, int64_t ld, int64_t* n_local_out, double* mu_host) {
  if (!s || !X) return set_error(c, PPCA_ERR_INVALID_ARG, "null spec or X");
  if (s->d < 1 || s->n_global < 1 || ld < s->d) return set_error(c, PPCA_ERR_INVALID_ARG, "bad n/d/ld");
  if ((ld * (int64_t)elt_size(s->dtype)) % 16 != 0) return set_error(c, PPCA_ERR_INVALID_ARG, "ld*elt must be 16B aligned");
  if (s->layout == PPCA_LAYOUT_INTERLEAVED) {
    if (s->block_rows < 1 || s->block_rows % c->world) return set_error(c, PPCA_ERR_INVALID_ARG, "world must divide block_rows");
    if ((s->n_global % s->block_rows) % c->world) return set_error(c, PPCA_ERR_INVALID_ARG, "world must divide the last block");
  }
  int64_t row0 = 0;
  int64_t n_local = local_rows(s, c->rank, c->world, &row0);
  RowMap rm{(int)s->layout, s->n_global, s->block_rows, row0, c->rank, c->world};
  double* mu = (double*)scratch(c, S_GEN3, (size_t)s->d * sizeof(double));
  if (!mu) return set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
  if (s->dtype == PPCA_F32_SPLIT && s->d % 8) return set_error(c, PPCA_ERR_INVALID_ARG, "PPCA_F32_SPLIT needs d %% 8 == 0");
  ppca_status st = s->dtype == PPCA_BF16 ? generate_t<__nv_bfloat16>(c, s, (__nv_bfloat16*)X, ld, n_local, rm, mu)
                                         : generate_t<float>(c, s, (float*)X, ld, n_local, rm, mu);
  if (st != PPCA_OK) return st;
  if (s->dtype == PPCA_F32_SPLIT) PPCA_TRY(split_f32(c, X, n_local, s->d, ld));
  if (mu_host)
    PPCA_TRY(check_cuda(c, cudaMemcpyAsync(mu_host, mu, s->d * sizeof(double), cudaMemcpyDeviceToHost, c->stream),
                        "copy mean"));
  if (n_local_out) *n_local_out = n_local;
  return PPCA_OK;
}

// ----------------------------------------------------------------------------- fp32 → split layout
// Rows are staged through a scratch copy (the split row overwrites its own fp32 bytes), block of rows
// at a time; hi = RN_bf16(x), lo = RN_bf16(x − hi).
__global__ void split_rows_kernel(const float* __restrict__ src, int64_t rows, int64_t d, int64_t ld,
                                  __nv_bfloat16* __restrict__ dst) {
  const int64_t r = blockIdx.y;
  if (r >= rows) return;
  const float* s = src + r * ld;
  __nv_bfloat16* o = dst + r * ld * 2;      // row stride in bf16 = 2·ld
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < d; j += (int64_t)gridDim.x * blockDim.x) {
    const float x = s[j];
    const __nv_bfloat16 hi = __float2bfloat16_rn(x);
    o[j] = hi;
    o[d + j] = __float2bfloat16_rn(x - __bfloat162float(hi));
  }
}

ppca_status split_f32(Ctx* c, void* X, int64_t n_local, int64_t d, int64_t ld) {
  if (n_local < 0 || d < 1 || ld < d || (ld % 4) || (d % 8) || (n_local > 0 && !X) ||
      (reinterpret_cast<uintptr_t>(X) % 16))
    return set_error(c, PPCA_ERR_INVALID_ARG, "ppca_split_f32: need ld >= d, ld %% 4 == 0, d %% 8 == 0, aligned X");
  if (n_local == 0) return PPCA_OK;
  const int64_t row_bytes = ld * 4;
  const int64_t blk = std::max<int64_t>(1, std::min<int64_t>(n_local, ((int64_t)64 << 20) / row_bytes));
  float* tmp = (float*)scratch(c, S_GEN2, (size_t)blk * row_bytes);
  if (!tmp) return set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
  for (int64_t r0 = 0; r0 < n_local; r0 += blk) {
    const int64_t rows = std::min(blk, n_local - r0);
    uint8_t* base = (uint8_t*)X + r0 * row_bytes;
    PPCA_TRY(check_cuda(c, cudaMemcpyAsync(tmp, base, (size_t)rows * row_bytes, cudaMemcpyDeviceToDevice, c->stream),
                        "split stage"));
    for (int64_t y0 = 0; y0 < rows; y0 += 65535) {
      const int64_t ry = std::min<int64_t>(65535, rows - y0);
      dim3 grid((unsigned)std::min<int64_t>(ceil_div(d, 256), 64), (unsigned)ry);
      split_rows_kernel<<<grid, 256, 0, c->stream>>>(tmp + y0 * ld, ry, d, ld,
                                                    reinterpret_cast<__nv_bfloat16*>(base + y0 * row_bytes));
      PPCA_LAUNCH_CHECK(c, "split_rows_kernel");
    }
  }
  return PPCA_OK;
}

// ----------------------------------------------------------------------------- philox words (tests)
__global__ void philox_words_kernel(uint64_t seed, uint32_t stream, uint64_t first, int64_t count, uint32_t* out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) out[i] = philox_word(seed, stream, first + (uint64_t)i);
}

ppca_status philox_words(Ctx* c, uint64_t seed, uint32_t stream, uint64_t first, int64_t count, uint32_t* out) {
  if (count <= 0) return PPCA_OK;
  philox_words_kernel<<<(unsigned)ceil_div(count, 256), 256, 0, c->stream>>>(seed, stream, first, count, out);
  PPCA_LAUNCH_CHECK(c, "philox_words");
  return PPCA_OK;
}

}  // namespace ppca
