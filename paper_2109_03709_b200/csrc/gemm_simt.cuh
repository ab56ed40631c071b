// gemm_simt.cuh — CUDA-core (fp32 FMA) streaming products over X, the first correct path.
//
// NT:  C[M][N] = A[M][K] · B[N][K]ᵀ        Y = X·Wᵀ      (M = rows, N = m, K = d)
// TN:  P[z][M][N] = Σ_{k ∈ split z} A[k][M] · B[k][N]   Z = YᵀX, S = YᵀY  (K = rows, split-K)
// The TN kernel accumulates each 16-row slab in fp32 and adds it to fp64 accumulators, so a
// sum over 10^6 rows keeps ~1e-7 relative accuracy; the split-K partials are reduced in a
// fixed order (deterministic, no atomics).
#pragma once
#include "common.cuh"

namespace ppca {

template <typename TX>
ppca_status launch_nt(Ctx* c, const TX* A, int64_t lda, const float* B, int64_t ldb, float* C,
                      int64_t ldc, int64_t M, int64_t N, int64_t K);

// P has room for nsplit * M * N doubles; returns nsplit used.
template <typename TA, typename TB>
ppca_status launch_tn_splitk(Ctx* c, const TA* A, int64_t lda, const TB* B, int64_t ldb,
                             double* P, int64_t M, int64_t N, int64_t K, int nsplit);

int tn_pick_splits(Ctx* c, int64_t M, int64_t N, int64_t K);

// out[i] = Σ_z P[z][i] (fixed order); out as float or double.  alpha scales the result.
ppca_status launch_reduce_splits_f32(Ctx* c, const double* P, int nsplit, int64_t count, float* out,
                                     int64_t ldo, int64_t cols);
ppca_status launch_reduce_splits_f64(Ctx* c, const double* P, int nsplit, int64_t count, double* out);
ppca_status launch_reduce_splits_f64(Ctx* c, const double* P, int nsplit, int64_t count, double* out,
                                     cudaStream_t st);

}  // namespace ppca
