/*
 * ppca.h — C ABI of the B200-native primed-PCA (pPCA) hot path (arXiv 2109.03709).
 *
 * The problem statement is Algorithm 1 of the paper: a centred dataset
 * X ∈ R^{n×d} (L14), parameters k, l and a PRIMING method in; the first k principal
 * directions (eigenvectors of XᵀX, L15) and their eigenvalue estimates out.  PRIMING
 * runs on m = k + l directions (§3.3 "Extra components", L111-114).
 *
 * Conventions (all entry points):
 *  - Vector sets are [m][d] row-major float32 device arrays: row i is the d-vector v_i
 *    ("ordered list of d-vectors").  X is row-major [n_local][ld] (float32 or bf16).
 *  - Ownership: the caller allocates every device buffer it passes (X, W, V, velocity, E, T)
 *    and every host output; the library never frees caller memory.  The context owns its
 *    NCCL communicator, its events and a grow-only device scratch pool.
 *  - Streams: all work is enqueued on the context's stream.  Each call synchronises that
 *    stream once before returning, so it can report a status; no host sync happens inside
 *    an iteration loop.
 *  - Collectives: with world > 1 every call is collective (like NCCL): all ranks call it with
 *    the same arguments except their own X shard; results (W, E, θ) are bitwise identical on
 *    all ranks.  The only collective is an NCCL all-reduce (sum) of per-rank partial products.
 *  - Errors: a non-OK status leaves outputs unspecified.  ppca_last_error() returns a message.
 *  - Numerics: X in fp32 or bf16; products accumulated in fp32 (hybrid fp32/fp64 for long
 *    reductions), every m×m quantity (Gram, Cholesky, Jacobi) in fp64.
 */
#ifndef PPCA_H
#define PPCA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PPCA_ABI_VERSION 1
#define PPCA_UNIQUE_ID_BYTES 128   /* sizeof(ncclUniqueId) */
#define PPCA_MAX_M 128             /* largest supported m = k + l */

typedef enum {
  PPCA_OK = 0,
  PPCA_ERR_INVALID_ARG = 1,          /* null pointer, bad enum, k > m, ld*elt % 16 != 0 ... */
  PPCA_ERR_DIM_MISMATCH = 2,
  PPCA_ERR_TOO_MANY_COMPONENTS = 3,  /* m > d or m > PPCA_MAX_M */
  PPCA_ERR_NONFINITE = 4,            /* a priming update produced Inf/NaN */
  PPCA_ERR_DEGENERATE = 5,           /* EigenGame v_iᵀMv_i <= 1e-12·max, zero vector (L225) */
  PPCA_ERR_SUBSPACE_COLLAPSE = 6,    /* orthonormalisation lost rank / fewer than k survive */
  PPCA_ERR_NO_CONVERGENCE = 7,       /* Jacobi exceeded 100 sweeps */
  PPCA_ERR_CUDA = 8,
  PPCA_ERR_NCCL = 9,
  PPCA_ERR_UNSUPPORTED = 10          /* not an sm_100 device, NCCL missing for world > 1, ... */
} ppca_status;

/* Storage of X.  PPCA_F32_SPLIT is the tensor-core-native layout of fp32 data: each fp32 value x is
 * held as the round-to-nearest bf16 pair hi = RN(x), lo = RN(x − hi) (x − (hi + lo) ≤ 2^-17·|x|,
 * unbiased), and row r of a shard [n_local][ld] (ld in 4-byte logical elements, ld ≥ d) holds the d hi
 * values followed by the d lo values (2·d bf16 = 4·d bytes, so the row is exactly as long as its fp32
 * form; d % 8 == 0 keeps the lo plane 16-byte aligned).  TMA stages both planes straight into the
 * UMMA swizzle and the X·Wᵀ product reads X_hi + X_lo, while the Xᵀ·Y product reads only the hi plane
 * (DESIGN.md §5), so no CUDA-core conversion runs per pass.  ppca_split_f32 converts fp32 rows in
 * place; ppca_generate writes it directly. */
typedef enum { PPCA_F32 = 0, PPCA_BF16 = 1, PPCA_F32_SPLIT = 2 } ppca_dtype;

/* Row layout of a shard.  CONTIGUOUS: rank g holds global rows [⌈n/G⌉g, ⌈n/G⌉(g+1)).
 * INTERLEAVED: every minibatch block of block_rows rows (the last one may be shorter, size p)
 * is split in G equal slices; rank g holds rows [s·b + g·p/G, s·b + (g+1)·p/G) of block s,
 * so a global minibatch is identical for every G (reading R10). */
typedef enum { PPCA_LAYOUT_CONTIGUOUS = 0, PPCA_LAYOUT_INTERLEAVED = 1 } ppca_layout;

typedef enum { PPCA_PLANTED_QR = 0, PPCA_PLANTED_HOUSEHOLDER = 1, PPCA_IMAGE_FACTOR = 2 } ppca_family;
typedef enum { PPCA_SPECTRUM_EXP = 0, PPCA_SPECTRUM_POWER = 1 } ppca_spectrum;

typedef struct ppca_ctx ppca_ctx;

/* This rank's row shard of the centred X. */
typedef struct {
  const void* data;     /* device, row-major [n_local][ld] of dtype */
  ppca_dtype dtype;
  int64_t n_local;      /* rows stored on this rank (may be 0) */
  int64_t n_global;     /* rows over all ranks */
  int64_t d;            /* dimension */
  int64_t ld;           /* row stride in elements, ld >= d, ld*sizeof(dtype) % 16 == 0 */
  ppca_layout layout;
  int64_t block_rows;   /* minibatch block b for INTERLEAVED (0 otherwise) */
} ppca_matrix;

/* Synthetic generator (BASELINE.json configs[0..4]). */
typedef struct {
  ppca_family family;
  ppca_spectrum spectrum;  /* EXP: λ_j = exp(-j/a); POWER: λ_j = j^-a; j = 1..d */
  double a;
  double noise;            /* added to every λ_j */
  int32_t relu;            /* planted_householder: max(0, ·) */
  int32_t house_r;         /* number of Householder reflections */
  int32_t rank;            /* image_factor inner dimension (50) */
  ppca_dtype dtype;        /* storage */
  int64_t n_global;
  int64_t d;
  uint64_t seed;
  ppca_layout layout;
  int64_t block_rows;
} ppca_gen_spec;

/* ---------------------------------------------------------------- context */
const char* ppca_status_string(ppca_status s);
int ppca_abi_version(void);

/* NCCL unique id for a world > 1 context (rank 0 calls it and broadcasts the bytes).
 * uid_out: host buffer of PPCA_UNIQUE_ID_BYTES. */
ppca_status ppca_get_unique_id(void* uid_out);

/* device: CUDA ordinal; stream: cudaStream_t or NULL (legacy default stream);
 * uid: PPCA_UNIQUE_ID_BYTES host bytes, required if world > 1.  With world == 1 a non-NULL uid creates a
 * one-rank NCCL communicator, so the collective call sites run on one GPU as well (tests); NULL: none.
 * Errors: INVALID_ARG, UNSUPPORTED (not sm_100 / NCCL missing), NCCL (CommInitRank failed or the
 * communicator's rank count differs from world), CUDA. */
ppca_status ppca_ctx_create(int device, void* stream, const void* uid, int rank, int world,
                            ppca_ctx** out);
ppca_status ppca_ctx_destroy(ppca_ctx* ctx);
/* Copies the last error message of ctx (NUL-terminated, truncated to cap). */
ppca_status ppca_last_error(const ppca_ctx* ctx, char* msg, size_t cap);
/* Number of library kernel launches enqueued by this context since creation (bench evidence). */
int64_t ppca_launch_count(const ppca_ctx* ctx);
/* Number of NCCL operations (one grouped [Z|S] all-reduce counts once) enqueued since creation. */
int64_t ppca_collective_count(const ppca_ctx* ctx);
/* 1 if this build reads experiment switches from the environment (-DPPCA_EXPERIMENTS), 0 for the
 * shipped library (bench.py asserts 0: no environment variable can change or skip its work). */
int ppca_experiments_enabled(void);

/* ---------------------------------------------------------------- hot path */

/* Writes this rank's shard of the seeded synthetic X (centred by the fp64 mean over all
 * n_global rows, rounded to spec->dtype; PPCA_F32_SPLIT = the fp32 values in split layout) into the
 * caller's device buffer X [n_local][ld].
 * n_local_out: rows written; col_mean_host: optional host double[d] receiving the mean. */
ppca_status ppca_generate(ppca_ctx* ctx, const ppca_gen_spec* spec, void* X, int64_t ld,
                          int64_t* n_local_out, double* col_mean_host);

/* In-place conversion of an fp32 shard [n_local][ld] (ld ≥ d, ld % 4 == 0, d % 8 == 0) into the
 * PPCA_F32_SPLIT layout (same buffer, same ld).  Bit-exact: hi = RN_bf16(x), lo = RN_bf16(x − hi). */
ppca_status ppca_split_f32(ppca_ctx* ctx, void* X, int64_t n_local, int64_t d, int64_t ld);

/* Host → device upload of a block of X's rows (the end-to-end path: the user's data lives in host memory;
 * P L14 "data X" in, no other preprocessing).  host: `rows` rows of X's logical element type with row stride
 * ld_host elements — fp32 for PPCA_F32 and PPCA_F32_SPLIT, bf16 for PPCA_BF16 — pinned (asynchronous on the
 * context stream) or pageable (staged by the driver).  They land in the device shard described by X at local
 * row r0 (0 ≤ r0, r0 + rows ≤ X->n_local); for PPCA_F32_SPLIT the fp32 rows are then split in place into the
 * bf16 hi / lo planes (bit-exact, as ppca_split_f32).  The host buffer must stay valid until the next call
 * that synchronises the context stream (every ABI call with host outputs does).  Errors: INVALID_ARG for a
 * NULL pointer or a row range outside the shard; CUDA for a failed copy. */
ppca_status ppca_upload_rows(ppca_ctx* ctx, const void* host, int64_t rows, int64_t ld_host, const ppca_matrix* X,
                             int64_t r0);

/* Block power priming (§2.1, multi-component by re-orthonormalisation L63):
 * per iteration Y = X·Wᵀ, Z = YᵀX (fused streaming pass over X), all-reduce, W ← orth(Z)
 * (Q-factor with positive diag R).  W: device [m][d] in/out.  init_seed != 0 initialises W
 * from N(0,1) draws (Philox stream 6) then orthonormalises; init_seed == 0 resumes from W.
 * iters: the iteration budget (BASELINE fixes 20/50/30, reading R13).
 * eps > 0: the paper's stop rule "terminates when ‖x_i − x_{i+1}‖ < ε" (P L61-62), applied to the
 * block as max_j ‖w_j^{t+1} − s_j w_j^t‖ < eps with s_j = sign⟨w_j^{t+1}, w_j^t⟩ (columns are defined up
 * to sign); checking it costs one host synchronisation per iteration.  eps <= 0: run all iters.
 * theta_hist_host: optional host double[iters*m]: row t holds the pPCA (Rayleigh–Ritz)
 * eigenvalue estimates of span(W_t) computed from the same pass (S_t = YᵀY), descending; rows past
 * the stop are zero.  iters_done (optional): iterations run. */
ppca_status ppca_prime_power(ppca_ctx* ctx, const ppca_matrix* X, int m, int iters, double eps,
                             uint64_t init_seed, float* W, double* theta_hist_host, int* iters_done);

/* Generalised Oja / Sanger minibatch priming (§2.2; Nesterov L326):
 * G = X_bᵀY_b − W·triu(Y_bᵀY_b) summed over the global minibatch (reading R8), v ← μv + G,
 * W ← W + α(G + μv).  Minibatch s uses global block s mod ⌈n/b⌉ (reading R10).
 * W, velocity: device [m][d] in/out; step_io: in = first global step, out = next step.
 * init_seed != 0 initialises W (unit N(0,1) rows) and zeroes velocity. */
ppca_status ppca_prime_oja(ppca_ctx* ctx, const ppca_matrix* X, int m, int batch, double alpha,
                           double momentum, int64_t steps, uint64_t init_seed, float* W,
                           float* velocity, int64_t* step_io);

/* α-EigenGame minibatch priming (§2.3 Eqs. 1-3; update rule reading R11):
 * ∇_j = 2M_b v_j − 2Σ_{i<j}(v_jᵀM_b v_i / v_iᵀM_b v_i) M_b v_i, tangent projection,
 * Nesterov, renormalisation.  Same argument conventions as ppca_prime_oja (V in/out). */
ppca_status ppca_prime_eigengame(ppca_ctx* ctx, const ppca_matrix* X, int m, int batch,
                                 double alpha, double momentum, int64_t steps,
                                 uint64_t init_seed, float* V, float* velocity,
                                 int64_t* step_io);

/* pPCA refinement, Algorithm 1 steps 2-5: B = orth(V); S = (XBᵀ)ᵀ(XBᵀ)
 * (projected covariance, never forming π_S(x)); (θ, U) = eig(S) in fp64 (generalised with
 * the Gram of the operand actually used); E = U_kᵀB with the sign convention (largest-|entry|
 * positive).  V: device [m][d]; E: device [k][d] out; theta_host: host double[k] out
 * (eigenvalues of XᵀX restricted to span V, unnormalised, descending); subspace_dim: out. */
ppca_status ppca_refine(ppca_ctx* ctx, const ppca_matrix* X, const float* V, int m, int k,
                        float* E, double* theta_host, int* subspace_dim);

/* ppca_refine with flags.  PPCA_REFINE_ORTHONORMAL: the caller guarantees that the rows of V are orthonormal
 * to fp32 rounding (e.g. the W returned by ppca_prime_power), so B = orth(V) is skipped (B = V; the Rayleigh–
 * Ritz step uses the Gram of the operand rows, so θ and E stay those of span V); no rank check is made. */
#define PPCA_REFINE_ORTHONORMAL 1u
ppca_status ppca_refine_ex(ppca_ctx* ctx, const ppca_matrix* X, const float* V, int m, int k, unsigned flags,
                           float* E, double* theta_host, int* subspace_dim);

/* Row-subsampled pPCA refinement (§5.2: "we only project 10% of the data for computing
 * full-PCA"; reading R25): as ppca_refine, but the projected covariance
 * is formed from the 128-row tiles of each shard whose Philox4x32-10 uniform (sample_seed, stream 7,
 * key = the global index of the tile's first row for CONTIGUOUS shards; tiles are cut from each shard's
 * first row) is below `fraction`, and θ are rescaled by
 * n_global / rows used (an estimate of XᵀX's eigenvalues).  fraction ≥ 1 is ppca_refine.
 * rows_used (optional): rows in the sample over all ranks.  An empty sample is INVALID_ARG. */
ppca_status ppca_refine_sampled(ppca_ctx* ctx, const ppca_matrix* X, const float* V, int m, int k,
                                double fraction, uint64_t sample_seed, float* E, double* theta_host,
                                int* subspace_dim, int64_t* rows_used);

/* Proposition 3 checker (§4.2 Prop. 3: "π_S(e_i) maximises Var on the orthogonal
 * complement of span(π_S(e_1),…)"; reading R28).
 * S = span V (orthonormalised as ppca_refine does, same drop rule); t_i = row i of T (the true
 * eigenvectors).  Condition i: the top eigenvector u_i of the projected covariance restricted to the
 * complement, within S, of span(π_S(t_1),…,π_S(t_{i−1})) is within angle `tol` of π_S(t_i).
 * X: as ppca_refine (world > 1: row shards, the projected Gram is all-reduced); V: device [m][d];
 * T: device [upto][d] fp32, upto ≤ PPCA_MAX_M; angles_host: host double[upto] out, ∠(u_i, π_S(t_i)) in
 * [0, π/2]; flags_host: host int[upto] out, 1 iff conditions 1 … i all hold (the chain breaks at the
 * first failure).  Errors: DEGENERATE if ‖π_S(t_i)‖ < 1e-10‖t_i‖, SUBSPACE_COLLAPSE if
 * dim S < upto, INVALID_ARG for null pointers, upto out of range or tol < 0.  Synchronises the stream.
 * Accuracy: S is spanned by fp32 rows, so angles below ~1e-6 are not resolved (tol is the caller's). */
ppca_status ppca_check_prop3(ppca_ctx* ctx, const ppca_matrix* X, const float* V, int m, const float* T,
                             int upto, double tol, double* angles_host, int* flags_host);

/* Theorem 1 as an online assertion (§4.2 Theorem 1 L308-312 with Prop. 3; SURVEY §8(f)
 * NEXT-4): call at a priming checkpoint with the priming output V (device [m][d]; its first k rows, normalised,
 * are e_i^PRIMING) and the true eigenvectors T (device [k][d]).  upto_out: length of the leading run of Prop. 3
 * conditions that hold within `tol` (as ppca_check_prop3).  On that run pPCA's i-th vector is the vector of
 * span V closest to e_i, so the theorem's conclusion is ∠(pPCA_i, e_i) ≤ ∠(e_i^PRIMING, e_i) (+ tol) —
 * hence LCES(pPCA) ≥ LCES(priming) for every threshold.  ang_priming_host / ang_ppca_host: host double[k] out;
 * holds_out: 1 iff the conclusion holds on the run (0 flags a violation).  Two passes over X (the checker's
 * projected Gram and the refine).  Errors: as ppca_check_prop3 and ppca_refine. */
ppca_status ppca_check_theorem1(ppca_ctx* ctx, const ppca_matrix* X, const float* V, int m, int k, const float* T,
                                double tol, int* upto_out, double* ang_priming_host, double* ang_ppca_host,
                                int* holds_out);

/* Evaluation (§5.3): angle_i = arccos(min(1,|<E_i,T_i>|)) and
 * LCES(V) = #consecutive i from 1 with angle_i < V (strict), for each threshold.
 * E, T: device [k][d] unit rows.  angles_host: double[k]; lces_host: int[nthr]. */
ppca_status ppca_eval(ppca_ctx* ctx, const float* E, const float* T, int k, int64_t d,
                      const double* thr_host, int nthr, double* angles_host, int* lces_host);

/* Certification support for the reference of large configs (reading R29):
 * res_host[i] = ‖XᵀX e_i − θ_i e_i‖₂ for the k rows e_i of E (device [k][d] fp32, unit rows) and
 * theta_host[i] (host double[k]).  By Weyl some eigenvalue of XᵀX lies within res_i of θ_i; with a gap δ
 * the angle to the true eigenvector is ≤ res_i/δ (Davis–Kahan).  One exact-fp32 CUDA-core pass over X
 * (no bf16 rounding of E or of X·Eᵀ), fp64 split-K sums, summed over ranks.  res_gram_host (optional, host
 * double[k*k]): the Gram R·Rᵀ of the residual rows, so ‖R‖₂ = sqrt(λ_max) for the sinΘ bound ‖R‖₂/δ.  Untimed
 * support, not a step of the method.  Errors: INVALID_ARG (null pointers), as ppca_refine for X, k ≤ min(d, 128). */
ppca_status ppca_ritz_residuals(ppca_ctx* ctx, const ppca_matrix* X, const float* E, int k,
                                const double* theta_host, double* res_host, double* res_gram_host);

/* Captured variance vᵀ(XᵀX)v = ‖Xv‖² for each row of V (PAPER.md L416 footnote),
 * summed over ranks.  var_host: double[m]. */
ppca_status ppca_captured_variance(ppca_ctx* ctx, const ppca_matrix* X, const float* V, int m,
                                   double* var_host);

/* Support (ground truth for evaluation, untimed): G = XᵀX in fp64, device double[d][d],
 * summed over ranks. */
ppca_status ppca_gram(ppca_ctx* ctx, const ppca_matrix* X, double* G);

/* Support (generator parity tests): Philox4x32-10 words w[e], e in [first, first+count) of
 * (seed, stream) into device uint32 out[count] (DESIGN.md §Inputs counter convention). */
ppca_status ppca_philox_words(ppca_ctx* ctx, uint64_t seed, uint32_t stream, uint64_t first,
                              int64_t count, uint32_t* out);

/* Timing hook (bench.py): with enable != 0, every streaming pass over X (power or refine
 * mode) is bracketed by CUDA events on the context stream.  ppca_get_pass_time returns the
 * summed device time (ms) and the number of passes recorded since the last call, then resets. */
ppca_status ppca_set_timing(ppca_ctx* ctx, int enable);
ppca_status ppca_get_pass_time(ppca_ctx* ctx, double* ms_total, int64_t* passes);

/* Timing hook (bench.py roofline of the dominant kernel): with timing enabled, each launch of the
 * tensor-core kernel A (which = 0: Y = X·W'ᵀ, S = YᵀY) and kernel B (which = 1: Zᵀ = XᵀY) is bracketed by
 * CUDA events on the context stream; returns the summed device time (ms) and launch count, then resets. */
ppca_status ppca_get_kernel_time(ppca_ctx* ctx, int which, double* ms_total, int64_t* launches);

/* Timing hook: select the fused-pass implementation (0 = auto, 1 = SIMT fp32, 2 = tcgen05, 3 = tcgen05
 * with the power pass as two kernels instead of a single-read fused kernel, 4 = tcgen05 with the power pass
 * on the row-group fused kernel (round 1) instead of the d-sliced pair kernel; 3 and 4 report as 2).
 * Returns UNSUPPORTED if the requested path cannot run this matrix. */
ppca_status ppca_set_pass_impl(ppca_ctx* ctx, int impl);
/* Re-orthonormalisation of the power iteration: 0 = auto — with world > 1 and d·m² ≥ 2^28 (C5)
 * the CholQR is split by d-slices (reduce-scatter of Z, slice Gram, m×m all-reduce, slice apply, all-gather of
 * W) so the d·m² work per rank drops by the rank count; 1 = replicated on every rank; -1 = the split path over
 * the context's ranks even at world 1 (needs a communicator; tests); b ≥ 2 at world 1 = b emulated slices
 * without NCCL (tests).  The result is the same CholQR (the Gram summed in another order). */
ppca_status ppca_set_orth_split(ppca_ctx* ctx, int split);
/* Implementation used by the most recent pass (1 = SIMT, 2 = tcgen05; 0 = none yet). */
int ppca_last_pass_impl(const ppca_ctx* ctx);
/* Kernels of the most recent tensor-core power pass (bench.py's roofline label): 2 = kernel A2 + kernel B
 * (X read twice), 3 = the row-group single-read kernel (xwz_fused_kernel), 4 = the d-sliced pair single-read
 * kernel (xwz_pair_kernel); 0 = none yet. */
int ppca_last_power_kernel(const ppca_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* PPCA_H */
