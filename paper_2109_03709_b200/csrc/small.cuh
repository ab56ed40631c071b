// small.cuh — the m×m side of the hot path: vector Gram, Cholesky-QR re-orthonormalisation,
// single-CTA fp64 Jacobi Rayleigh–Ritz, rotation, sign convention, priming updates.
#pragma once
#include "common.cuh"

namespace ppca {

// G[m][m] (fp64) = V Vᵀ for row vectors V [m][d] fp32 (partials in S_PART).
ppca_status vec_gram(Ctx* c, const float* V, int m, int64_t d, double* G);
// the same on stream st with its split partials in scratch slot part_slot (side-stream use)
ppca_status vec_gram_on(Ctx* c, const float* V, int m, int64_t d, double* G, cudaStream_t st, int part_slot);
size_t vec_gram_part_bytes(const Ctx* c, int m, int64_t d);
// Linv = chol(G)⁻¹ (lower, fp64, one CTA) on stream st; row_map/m_out as in cholqr (no drops)
ppca_status chol_inv_on(Ctx* c, const double* G, int m, double* Linv, int* row_map, int* m_out, cudaStream_t st);
// OUT = L·IN, L lower-triangular fp64 m×m, IN/OUT [m][d] fp32 (distinct buffers)
ppca_status apply_lower_on(Ctx* c, const double* L, int m, const float* IN, int64_t d, float* OUT, cudaStream_t st);

// CholQR2 in place: W [m][d] ← Q-factor of the rows (positive diag R), twice.
// drop_tol > 0: rows whose Cholesky pivot ≤ drop_tol²·G_jj are dropped (refine semantics,
// SPEC L51); the survivors are compacted to the front, *m_out receives their count.
// drop_tol == 0: any non-positive pivot flags SUBSPACE_COLLAPSE (power-iteration semantics).
ppca_status cholqr2(Ctx* c, float* W, int m, int64_t d, double drop_tol, int* m_out);
// General form: W (may alias Zin) = orth(Zin) with `passes` Cholesky-QR passes.
// The power loop's next pass operand W' = [W_hi; W_lo] (bf16 rows hi = RN(W), lo = RN(W − hi), lo rows at
// lo_off elements) and Wr = hi + lo, written by CholQR's apply together with W (what prep_w would compute
// from W, bit for bit) when wprep_fusable(): one launch fewer per power iteration.
struct WPrep {
  __nv_bfloat16* Wb;
  float* Wr;
  int64_t lo_off;
};
bool wprep_fusable(const Ctx* c, int m, int mp, int64_t d);
// gram_ready: the S_GRAM scratch already holds ZinᵀZin (the power pass's reduce_zp_gram; one pass, no drops)
ppca_status cholqr(Ctx* c, const float* Zin, float* W, int m, int64_t d, double drop_tol, int* m_out, int passes,
                   bool gram_ready = false, const WPrep* prep = nullptr);

// Rayleigh–Ritz in one CTA (fp64): given S = (XWᵀ)ᵀ(XWᵀ) and Bm = WWᵀ of the operand rows,
// solve S u = θ Bm u:  L = chol(Bm), Jacobi(L⁻¹SL⁻ᵀ) → θ (desc), U;  R = Uᵀ L⁻¹.
// theta_dev: double[m]; R_dev: double[m][m] (row i lifts eigenvector i: e_i = Σ_j R_ij w_j).
ppca_status ritz_solve(Ctx* c, const double* S, const double* Bm, int m, double* theta_dev,
                       double* R_dev, cudaStream_t stream, int top = 0);   // top > 0: only the top largest pairs (R_dev)

// E[k][d] = R[:k] · W  (fp64 accumulate), then the sign convention on each row.
ppca_status lift_rows(Ctx* c, const double* R, int ldr, const float* W, int m, int k, int64_t d,
                      float* E, bool apply_sign, cudaStream_t stream);

// W[c][j] = N(0,1) draw (seed, stream 6, c·d + j), rows scaled to unit norm.
ppca_status init_rows(Ctx* c, uint64_t seed, float* W, int m, int64_t d);
// rows scaled to unit norm (fp64 norms); flags DEGENERATE on a zero row.
ppca_status normalize_rows(Ctx* c, float* W, int m, int64_t d);

// Oja / Sanger update (fp64 per element):  G = Q − tril(P)·W;  v ← μv + G;  W ← W + α(G + μv).
ppca_status oja_update(Ctx* c, const float* Q, const double* P, float* W, float* vel, int m,
                       int64_t d, double alpha, double mu);
// Generalized Oja, all `steps` steps in one cooperative kernel (oja_persistent.cu): single GPU, m ≤ 64,
// short windows, automatic pass selection.  Returns false (nothing launched) when not applicable.
bool oja_persistent(Ctx* c, const ppca_matrix* X, int m, int batch, double alpha, double mu, int64_t s0,
                    int64_t steps, float* W, float* vel, ppca_status* st);
// EigenGame update: coefficients from A, r = 2MV − 2 N·MV − 2U∘V, Nesterov, renormalise.
// prep: also write the next window pass's operand split of V (prep_done: it was written — the fused kernel ran)
ppca_status eigengame_update(Ctx* c, const float* MV, const double* A, float* V, float* vel, int m,
                             int64_t d, double alpha, double mu, const WPrep* prep = nullptr, bool* prep_done = nullptr);

// dots[i] = <E_i, T_i> in fp64.
// Prop. 3 checker (reading R28): from the stacked Gram G ([B; T], ld g) and S, the angles between π_S(t_i)
// and the top eigenvector of the projected covariance on the complement of π_S(t_1..t_{i−1}); the ratios
// ‖π_S(t_i)‖/‖t_i‖ come back first (DEGENERATE below 1e-10).  Synchronises the stream.
ppca_status prop3_device(Ctx* c, const double* G, int g, const double* S, int mm, int upto, double* ratio_host,
                         double* angles_host);
ppca_status row_dots(Ctx* c, const float* E, const float* T, int k, int64_t d, double* dots);
// res[i] = ‖Z_i − θ_i E_i‖ (fp64), θ device double[k]
ppca_status ritz_resid(Ctx* c, const float* Z, const float* E, const double* theta, int k, int64_t d, double* res);
// Z_i ← Z_i − θ_i E_i in place
ppca_status resid_rows(Ctx* c, float* Z, const float* E, const double* theta, int k, int64_t d);

}  // namespace ppca
