// common.cuh — shared internals of libppca (context, errors, scratch, Philox, small helpers).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string>
#include <vector>

#include "../../include/ppca.h"

namespace ppca {

// ----------------------------------------------------------------------------- device error word
// Kernels set bits here instead of trapping; the host reads it once per ABI call.
enum DevErr : int {
  DEV_OK = 0,
  DEV_NONFINITE = 1,
  DEV_DEGENERATE = 2,
  DEV_COLLAPSE = 4,
  DEV_NOCONV = 8,
  DEV_TIMEOUT = 16,     // a bounded inter-CTA wait expired (fused pass: CTAs not co-resident)
};

struct Ctx;
typedef ppca_status (*AllreduceFn)(Ctx*, void* buf, size_t count, int is_f64);

struct Ctx {
  int device = 0;
  int rank = 0, world = 1;
  cudaStream_t stream = nullptr;      // the library's stream (own high-priority stream, or the caller's)
  cudaStream_t user_stream = nullptr; // the caller's stream (ppca_ctx_create)
  bool own_stream = false;
  cudaEvent_t fork_ev = nullptr;      // caller's stream → library stream at every ABI entry
  cudaStream_t side = nullptr;        // side stream (Ritz solves overlap the next pass)
  cudaEvent_t prep_ev = nullptr;     // when set: recorded once the pass operand W' is prepared (power loop)
  // deferred S reduction of the fused pass (power loop with θ history on one GPU: S feeds only the side-stream
  // Ritz solve): the pass records s_ev_pass and leaves the partials; pass_reduce_deferred_s reduces them on a
  // given stream and records s_ev_red, which the next fused pass waits for before rewriting the partials
  bool s_defer = false;
  bool s_skip = false;                // power loop without θ history on one rank: the pass's S is not reduced
  bool s_pending = false;
  cudaEvent_t s_ev_pass = nullptr, s_ev_red = nullptr;
  const double* s_part = nullptr;
  int s_parts = 0, s_mp = 0, s_m = 0;
  // deferred Z reduction (EigenGame steps on one GPU): the window pass leaves its row-group partials and the
  // update kernel sums them while staging (pass_reduce_deferred_z reduces them for any other consumer)
  bool zp_defer = false, zp_pending = false;
  const float* zp_part = nullptr;
  int64_t zp_nrg = 0, zp_dpad = 0, zp_d = 0;
  int zp_mp = 0, zp_m = 0;
  bool side_busy = false;             // side-stream kernels may overlap the next pass: persistent
                                      // pass kernels then leave one SM free (a late CTA stalls the pass)
  cudaEvent_t ev_a = nullptr, ev_b = nullptr;
  void* nccl_comm = nullptr;          // ncclComm_t when world > 1
  int* d_err = nullptr;               // device error word
  int pass_impl = 0;                  // 0 auto, 1 simt, 2 tcgen05, 3 tcgen05 without the fused power pass
  int* flags = nullptr;               // per-tile ready flags of the fused power pass (device, zeroed)
  int64_t flags_n = 0;
  int epoch = 0;
  int last_impl = 0;                  // implementation of the most recent pass
  int last_power_kernel = 0;          // kernels of the most recent tensor-core power pass (ppca_last_power_kernel)
  int sm_count = 148;
  int64_t launches = 0;
  int64_t collectives = 0;            // NCCL operations enqueued (bench evidence of the exchange)
  // distributed CholQR (§6): 0 = auto, 1 = replicated, b ≥ 2 = d-slices (world == 1: b emulated slices, tests)
  int orth_split = 0;
  int64_t z_block_cols = 0;           // > 0: the pass writes Z d-blocked [d/z_block_cols][m][z_block_cols]
  // power loop on one rank (no later all-reduce of Z): the pass may also leave G = ZᵀZ (fp64, S_GRAM) for the
  // CholQR that follows (zgram_want: allowed; zgram_done: it did)
  bool zgram_want = false;
  bool zgram_done = false;
  // power loop: CholQR's apply already wrote the next pass operand W' of W = wprep_for (prep_w adopts it)
  const float* wprep_for = nullptr;
  __nv_bfloat16* wprep_b = nullptr;
  float* wprep_r = nullptr;
  // pass timing (bench): event pairs recorded around each pass
  bool timing = false;
  std::vector<cudaEvent_t> tev;
  size_t tev_used = 0;
  // per-kernel timing of the tensor-core pass kernels: [0] kernel A (Y = XW'ᵀ, S), [1] kernel B (Zᵀ = XᵀY)
  std::vector<cudaEvent_t> kev[2];
  size_t kev_used[2] = {0, 0};
  std::string last_error;
  // grow-only scratch slots
  static const int kSlots = 32;
  void* slot_ptr[kSlots] = {};
  size_t slot_bytes[kSlots] = {};
};

// scratch slot ids
enum Slot {
  S_PART = 0,    // split-K partials (fp64/fp32)
  S_Y,           // Y = X·Wᵀ (n_local × m)
  S_Z,           // Z (m × d) fp32
  S_S,           // S (m × m) fp64 (+ allreduce payload)
  S_GRAM,        // m×m fp64 gram of vectors
  S_SMALL,       // small fp64 work (L, Linv, U, R ...)
  S_W2,          // m × d fp32 temp
  S_W3,          // m × d fp32 temp
  S_ROWRED,      // per-row reductions
  S_GEN0, S_GEN1, S_GEN2, S_GEN3,  // generator buffers
  S_EVAL,
  S_TC0, S_TC1, S_TC2, S_TC3, S_TC4,   // tensor-core pass scratch
  S_TILES,                         // row-tile list of the subsampled refine (int32)
  S_SIDE,                          // side-stream m×m work of the power loop (Linv[2], row maps)
  S_SIDE_PART,                     // side-stream split partials (vector Gram)
  S_NTSTAGE,
  S_P3,                            // Prop. 3 checker workspace (fp64)
  S_P3F,                           // Prop. 3 checker stacked vectors [B; T] (fp32)
  S_EPS,                           // power stop rule: W_t copy + column dots
  S_DIST,                          // distributed CholQR: this rank's Z slice and W slice
  S_SIGN,                          // sign convention partials of very long rows
  S_ZGRAM,                         // cluster partials of the pass's Gram of Z (reduce_zp_gram)
  S_WPREP,                         // the power loop's second W' buffer (written by CholQR's apply)
};

void* scratch(Ctx* c, int slot, size_t bytes);     // grow-only, device memory

ppca_status set_error(Ctx* c, ppca_status s, const char* fmt, ...);
ppca_status check_cuda(Ctx* c, cudaError_t e, const char* what);
ppca_status finish(Ctx* c, const char* what);      // sync stream, read error word, map to status
ppca_status allreduce(Ctx* c, void* buf, size_t count, bool f64);
ppca_status allreduce_zs(Ctx* c, float* Z, size_t nz, double* S, size_t ns);   // grouped [Z | S]
ppca_status pass_reduce_deferred_z(Ctx* c, float* Z);   // Z from the partials a deferred pass left (no-op otherwise)

#define PPCA_TRY(expr)                         \
  do {                                         \
    ppca_status _s = (expr);                   \
    if (_s != PPCA_OK) return _s;              \
  } while (0)

#define PPCA_LAUNCH_CHECK(c, what)                                        \
  do {                                                                    \
    (c)->launches++;                                                      \
    cudaError_t _e = cudaGetLastError();                                  \
    if (_e != cudaSuccess) return check_cuda((c), _e, what);              \
  } while (0)

// Experiment switches (tuning sweeps, ablations, phase skips used while profiling): read from the
// environment only in a build compiled with -DPPCA_EXPERIMENTS.  The shipped library always takes the
// default, so no environment variable can change or skip its work (ppca_experiments_enabled() == 0).
static inline int tune_env(const char* name, int dflt) {
#ifdef PPCA_EXPERIMENTS
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
#else
  (void)name;
  return dflt;
#endif
}

// ----------------------------------------------------------------------------- programmatic dependent launch
// The m×m chain between two passes is a row of short dependent kernels; with stream serialisation each one
// starts only after its predecessor has drained, so every boundary costs a launch latency.  The chain kernels
// are launched with programmatic stream serialisation instead: the dependent grid may become resident while
// its predecessor still runs and blocks in pdl_wait() (griddepcontrol.wait: returns once every prerequisite
// grid has completed and its memory is visible) before it touches global memory; each kernel calls
// pdl_trigger() right after its own wait, so at most one grid waits behind a running one.  Both instructions
// are no-ops in a grid launched without the attribute, so every kernel may carry them.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_enter() {
  pdl_wait();
  pdl_trigger();
}

extern int g_pdl;   // 1: chain kernels use programmatic dependent launch (experiment builds: PPCA_PDL=0 turns it off)

template <typename... KArgs, typename... Args>
static inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                     Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = g_pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// cudaFuncSetAttribute (dynamic shared memory opt-in) belongs to each device's context: call sites keep a
// bit mask of the devices already configured and apply the attribute once per device.
static inline bool first_on_device(uint64_t* mask, int dev) {
  const uint64_t bit = 1ull << (dev & 63);
  if (*mask & bit) return false;
  *mask |= bit;
  return true;
}

static inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
static inline size_t elt_size(ppca_dtype t) { return t == PPCA_BF16 ? 2 : 4; }

// One logical element of a PPCA_F32_SPLIT row (4 bytes: pointer arithmetic p + r·ld lands on row r);
// the row holds d bf16 hi values then d bf16 lo values, x = hi + lo (exact in fp32).
struct SplitF32 {
  uint32_t raw;
};

// ----------------------------------------------------------------------------- element loads
__device__ __forceinline__ float load_elt(const float* p, int64_t i) { return p[i]; }
__device__ __forceinline__ float load_elt(const __nv_bfloat16* p, int64_t i) { return __bfloat162float(p[i]); }
// element (r, c) of a matrix whose rows hold `ncols` logical columns (ncols matters for SplitF32 only)
__device__ __forceinline__ float load_rc(const float* p, int64_t ld, int64_t r, int64_t c, int64_t) { return p[r * ld + c]; }
__device__ __forceinline__ float load_rc(const __nv_bfloat16* p, int64_t ld, int64_t r, int64_t c, int64_t) {
  return __bfloat162float(p[r * ld + c]);
}
__device__ __forceinline__ float load_rc(const SplitF32* p, int64_t ld, int64_t r, int64_t c, int64_t ncols) {
  const __nv_bfloat16* row = reinterpret_cast<const __nv_bfloat16*>(p + r * ld);
  return __bfloat162float(row[c]) + __bfloat162float(row[ncols + c]);
}

// ----------------------------------------------------------------------------- Philox4x32-10
// Salmon et al. (SC'11); identical to curand_Philox4x32_10.  Counter convention:
// ctr = (call_lo, call_hi, stream, 0), key = (seed_lo, seed_hi); element e uses word e % 4 of call e / 4.
__host__ __device__ __forceinline__ void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
    k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
  }
}

__host__ __device__ __forceinline__ uint32_t philox_word(uint64_t seed, uint32_t stream, uint64_t e) {
  uint64_t call = e >> 2;
  uint32_t c[4] = {(uint32_t)call, (uint32_t)(call >> 32), stream, 0u};
  philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
  return c[e & 3];
}

__host__ __device__ __forceinline__ double u32_to_unit(uint32_t w) { return ((double)w + 0.5) * 2.3283064365386963e-10; }

// Gaussian element e of a stream: Box–Muller on the word pair (2⌊e/2⌋, 2⌊e/2⌋+1).
__device__ __forceinline__ double gaussian_elt(uint64_t seed, uint32_t stream, uint64_t e) {
  uint64_t pair = e >> 1;
  uint64_t call = pair >> 1;
  uint32_t c[4] = {(uint32_t)call, (uint32_t)(call >> 32), stream, 0u};
  philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
  uint32_t w0 = (pair & 1) ? c[2] : c[0];
  uint32_t w1 = (pair & 1) ? c[3] : c[1];
  double u0 = u32_to_unit(w0), u1 = u32_to_unit(w1);
  double rad = sqrt(-2.0 * log(u0));
  double ang = 6.283185307179586 * u1;
  return (e & 1) ? rad * sin(ang) : rad * cos(ang);
}

__device__ __forceinline__ double exponential_elt(uint64_t seed, uint32_t stream, uint64_t e) {
  return -log(u32_to_unit(philox_word(seed, stream, e)));
}

// RNE fp64 → bf16 (bit trick on the fp64 significand; exact for the normal range).
__device__ __forceinline__ __nv_bfloat16 f64_to_bf16_rne(double x) {
  unsigned long long b = (unsigned long long)__double_as_longlong(x);
  unsigned long long lsb = (b >> 45) & 1ull;
  b = (b + ((1ull << 44) - 1ull) + lsb) & ~((1ull << 45) - 1ull);
  float f = (float)__longlong_as_double((long long)b);   // exact: 8 significant bits
  unsigned int u = __float_as_uint(f) >> 16;
  __nv_bfloat16_raw r;
  r.x = (unsigned short)u;
  return __nv_bfloat16(r);
}

// ----------------------------------------------------------------------------- reductions
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// s = Σ load(i) for i = begin, begin + step, … < end, added in exactly that order (bit-identical to the plain
// loop) but with U loads in flight before the adds: a plain accumulation loop waits a full L2/HBM round
// trip per term when the compiler does not hoist the loads.
template <int U, typename L>
__device__ __forceinline__ double sum_in_order(int64_t begin, int64_t end, int64_t step, L load) {
  double s = 0.0;
  int64_t i = begin;
  for (; i + (U - 1) * step < end; i += U * step) {
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = load(i + u * step);
#pragma unroll
    for (int u = 0; u < U; ++u) s += v[u];
  }
  if (i < end) {                                  // the tail as one more batch (loads in flight together)
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = i + u * step < end ? load(i + u * step) : 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i + u * step < end) s += v[u];           // same order as the loop it replaces
  }
  return s;
}

// store(e, load(e)) for e = first, first + stride, … < count with U loads in flight before the stores
// (out-of-range lanes of the last batch load element count − 1 and store nothing).
template <int U, typename L, typename S>
__device__ __forceinline__ void copy_batched(int64_t first, int64_t count, int64_t stride, L load, S store) {
  for (int64_t e0 = first; e0 < count; e0 += U * stride) {
    decltype(load(e0)) v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = e0 + u * stride;
      v[u] = load(e < count ? e : count - 1);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = e0 + u * stride;
      if (e < count) store(e, v[u]);
    }
  }
}

}  // namespace ppca
