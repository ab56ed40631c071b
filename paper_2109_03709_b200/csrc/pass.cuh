// pass.cuh — the streaming pass over X (§8 rows a2 / a7): one interface, two implementations.
//   impl 1 (SIMT):    Y = X·Wᵀ (CUDA-core tiles), then Z = YᵀX and S = YᵀY (split-K, fp32→fp64).
//   impl 2 (tcgen05): fused tensor-core pass (pass_tc.cu) — X staged once per tile.
#pragma once
#include "common.cuh"

namespace ppca {

struct PassPlan {
  int impl = 1;
  bool precise = false;         // product 2 also reads X_lo of a split X (minibatch steps: Q is the update)
  // refine-mode pass over a subset of 128-row tiles (row-subsampled refine): device and host lists
  const int32_t* tiles_dev = nullptr;
  const int32_t* tiles_host = nullptr;
  int64_t ntiles_sel = -1;      // < 0: all rows
  const float* Wop = nullptr;   // fp32 values of the operand rows the last pass actually used
                                // (W itself for SIMT; RN_bf16(W) for tcgen05) — for the Ritz Gram
};

ppca_status pass_prepare(Ctx* c, const ppca_matrix* X, int m, PassPlan* plan);
// power mode: Z[m][d] (fp32) = (X·Wᵀ)ᵀX over the local rows, S[m][m] (fp64) = (X·Wᵀ)ᵀ(X·Wᵀ)
ppca_status pass_power(Ctx* c, const ppca_matrix* X, const PassPlan* plan, const float* W, int m, float* Z, double* S);
// refine mode: S only
ppca_status pass_gram(Ctx* c, const ppca_matrix* X, const PassPlan* plan, const float* W, int m, double* S);
void pass_release(Ctx* c);
ppca_status pass_time_collect(Ctx* c, double* ms, int64_t* n);
// per-kernel CUDA events around the tensor-core kernels (which: 0 = kernel A, 1 = kernel B); a mark pair
// brackets one launch
void kernel_timer_mark(Ctx* c, int which);
ppca_status kernel_time_collect(Ctx* c, int which, double* ms, int64_t* n);

// building blocks (SIMT), local rows [r0, r0+rows)
ppca_status xw(Ctx* c, const ppca_matrix* X, int64_t r0, int64_t rows, const float* W, int m, float* Y);
ppca_status ytx(Ctx* c, const ppca_matrix* X, int64_t r0, int64_t rows, const float* Y, int m, float* Z);
ppca_status yty(Ctx* c, const float* Y, int m, int64_t rows, double* S);

// the fused pass's deferred S reduction (Ctx::s_defer) on stream st; no-op when nothing is pending
size_t zgram_part_bytes(int m, int64_t d);   // scratch S_ZGRAM of the power pass's fused Z Gram
ppca_status pass_reduce_deferred_s(Ctx* c, double* S, cudaStream_t st);

}  // namespace ppca
