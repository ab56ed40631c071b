// api.cu — the C ABI (include/ppca.h): context, NCCL plumbing, and the hot-path drivers.
#include <dlfcn.h>
#include <stdarg.h>
#include <math.h>
#include <cmath>
#include <algorithm>
#include <nccl.h>

#include "common.cuh"
#include "gemm_simt.cuh"
#include "small.cuh"
#include "pass.cuh"

struct ppca_ctx {
  ppca::Ctx c;
};

namespace ppca {

int g_pdl = tune_env("PPCA_PDL", 1);

// ABI entry: select the device and order the library stream after the caller's stream
static void enter(Ctx* c) {
  c->wprep_for = nullptr;                       // a fused operand split never outlives the call that wrote it
  c->s_skip = false;
  cudaSetDevice(c->device);
  if (c->own_stream) {
    cudaEventRecord(c->fork_ev, c->user_stream);
    cudaStreamWaitEvent(c->stream, c->fork_ev, 0);
  }
}

ppca_status generate(Ctx* c, const ppca_gen_spec* s, void* X, int64_t ld, int64_t* n_local_out, double* mu_host);
ppca_status philox_words(Ctx* c, uint64_t seed, uint32_t stream, uint64_t first, int64_t count, uint32_t* out);
ppca_status split_f32(Ctx* c, void* X, int64_t n_local, int64_t d, int64_t ld);
ppca_status debug_wait_counters(unsigned long long* out16);

// ----------------------------------------------------------------------------- NCCL (dlopen)
struct NcclApi {
  bool loaded = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
};
static NcclApi g_nccl;

static bool nccl_load() {
  if (g_nccl.loaded) return true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return false;
  g_nccl.GetUniqueId = (decltype(g_nccl.GetUniqueId))dlsym(h, "ncclGetUniqueId");
  g_nccl.CommInitRank = (decltype(g_nccl.CommInitRank))dlsym(h, "ncclCommInitRank");
  g_nccl.AllReduce = (decltype(g_nccl.AllReduce))dlsym(h, "ncclAllReduce");
  g_nccl.CommDestroy = (decltype(g_nccl.CommDestroy))dlsym(h, "ncclCommDestroy");
  g_nccl.GroupStart = (decltype(g_nccl.GroupStart))dlsym(h, "ncclGroupStart");
  g_nccl.GroupEnd = (decltype(g_nccl.GroupEnd))dlsym(h, "ncclGroupEnd");
  g_nccl.GetErrorString = (decltype(g_nccl.GetErrorString))dlsym(h, "ncclGetErrorString");
  g_nccl.CommGetAsyncError = (decltype(g_nccl.CommGetAsyncError))dlsym(h, "ncclCommGetAsyncError");
  g_nccl.CommCount = (decltype(g_nccl.CommCount))dlsym(h, "ncclCommCount");
  g_nccl.ReduceScatter = (decltype(g_nccl.ReduceScatter))dlsym(h, "ncclReduceScatter");
  g_nccl.AllGather = (decltype(g_nccl.AllGather))dlsym(h, "ncclAllGather");
  g_nccl.loaded = g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.AllReduce && g_nccl.CommDestroy;
  return g_nccl.loaded;
}

// ----------------------------------------------------------------------------- errors / scratch
ppca_status set_error(Ctx* c, ppca_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->last_error = buf;
  return s;
}

ppca_status check_cuda(Ctx* c, cudaError_t e, const char* what) {
  if (e == cudaSuccess) return PPCA_OK;
  return set_error(c, PPCA_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

void* scratch(Ctx* c, int slot, size_t bytes) {
  if (bytes == 0) bytes = 16;
  if (c->slot_bytes[slot] >= bytes) return c->slot_ptr[slot];
  if (c->slot_ptr[slot]) {
    cudaStreamSynchronize(c->stream);
    if (c->side) cudaStreamSynchronize(c->side);
    cudaFree(c->slot_ptr[slot]);
    c->slot_ptr[slot] = nullptr;
    c->slot_bytes[slot] = 0;
  }
  size_t want = bytes + bytes / 4;
  static int dbg = -1;
  if (dbg < 0) dbg = tune_env("PPCA_DEBUG_SCRATCH", 0);
  if (dbg) fprintf(stderr, "[ppca] scratch slot %d grows to %zu bytes\n", slot, want);
  void* p = nullptr;
  if (cudaMalloc(&p, want) != cudaSuccess) {
    cudaGetLastError();
    if (cudaMalloc(&p, bytes) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    want = bytes;
  }
  c->slot_ptr[slot] = p;
  c->slot_bytes[slot] = want;
  return p;
}

ppca_status finish(Ctx* c, const char* what) {
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e == cudaSuccess && c->side) e = cudaStreamSynchronize(c->side);
  if (e != cudaSuccess) return check_cuda(c, e, what);
  int h = 0;
  e = cudaMemcpy(&h, c->d_err, sizeof(int), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return check_cuda(c, e, what);
  if (h) cudaMemset(c->d_err, 0, sizeof(int));
  if (h & DEV_NONFINITE) return set_error(c, PPCA_ERR_NONFINITE, "%s: non-finite update", what);
  if (h & DEV_DEGENERATE) return set_error(c, PPCA_ERR_DEGENERATE, "%s: degenerate denominator / zero vector", what);
  if (h & DEV_COLLAPSE) return set_error(c, PPCA_ERR_SUBSPACE_COLLAPSE, "%s: orthonormalisation lost rank", what);
  if (h & DEV_NOCONV) return set_error(c, PPCA_ERR_NO_CONVERGENCE, "%s: Jacobi exceeded 100 sweeps", what);
  if (h & DEV_TIMEOUT)
    return set_error(c, PPCA_ERR_CUDA, "%s: an inter-CTA wait of the fused pass timed out (CTAs not co-resident)", what);
  if (c->nccl_comm && g_nccl.CommGetAsyncError) {       // a communicator that failed asynchronously (peer lost, ...)
    ncclResult_t ar = ncclSuccess;
    if (g_nccl.CommGetAsyncError((ncclComm_t)c->nccl_comm, &ar) != ncclSuccess || ar != ncclSuccess)
      return set_error(c, PPCA_ERR_NCCL, "%s: NCCL communicator error: %s", what, g_nccl.GetErrorString(ar));
  }
  return PPCA_OK;
}

// In-place sum over the ranks on the context stream — the only collective of the path (BASELINE north_star:
// "combined with NCCL allreduce").  A context without a communicator (world 1) skips it.
ppca_status allreduce(Ctx* c, void* buf, size_t count, bool f64) {
  if (!c->nccl_comm || count == 0) return PPCA_OK;
  ncclResult_t r = g_nccl.AllReduce(buf, buf, count, f64 ? ncclFloat64 : ncclFloat32, ncclSum,
                                    (ncclComm_t)c->nccl_comm, c->stream);
  if (r != ncclSuccess) return set_error(c, PPCA_ERR_NCCL, "ncclAllReduce: %s", g_nccl.GetErrorString(r));
  c->collectives++;
  return PPCA_OK;
}

// The per-iteration exchange [Z | S] (fp32 d×m and fp64 m×m) as ONE grouped NCCL operation (one launch,
// one synchronisation point), SURVEY §8(e) "one fused buffer per step".
ppca_status allreduce_zs(Ctx* c, float* Z, size_t nz, double* S, size_t ns) {
  if (!c->nccl_comm) return PPCA_OK;
  ncclResult_t r = g_nccl.GroupStart ? g_nccl.GroupStart() : ncclSuccess;
  if (r == ncclSuccess && nz)
    r = g_nccl.AllReduce(Z, Z, nz, ncclFloat32, ncclSum, (ncclComm_t)c->nccl_comm, c->stream);
  if (r == ncclSuccess && ns)
    r = g_nccl.AllReduce(S, S, ns, ncclFloat64, ncclSum, (ncclComm_t)c->nccl_comm, c->stream);
  ncclResult_t r2 = g_nccl.GroupEnd ? g_nccl.GroupEnd() : ncclSuccess;
  if (r != ncclSuccess || r2 != ncclSuccess)
    return set_error(c, PPCA_ERR_NCCL, "grouped ncclAllReduce [Z|S]: %s", g_nccl.GetErrorString(r != ncclSuccess ? r : r2));
  c->collectives++;
  return PPCA_OK;
}

// ----------------------------------------------------------------------------- distributed CholQR (§6)
// The replicated part of a power iteration is W ← orth(Z) on the full d×m Z (d·m² fp64 MAC in the Gram, d·m²/2
// in the apply) on every rank.  Split by d-slices instead: the pass writes Z d-blocked [G][m][ds] (ds = d/G,
// launch_reduce_zp), one grouped NCCL operation reduce-scatters the slices (rank g receives Σ_ranks Z[:, slice g])
// and all-reduces S; every rank forms its slice's Gram, the m×m Grams are all-reduced, every rank factors the
// same G = Σ_g G_g (Cholesky + L⁻¹, replicated, m×m), applies L⁻¹ to its slice, and an all-gather assembles W.
// Exchange volume equals the all-reduce's (reduce-scatter + all-gather), plus one m×m all-reduce; the d·m² work
// per rank drops by G.  Test modes on one GPU: split = -1 runs the NCCL path with world's ranks (one-rank
// communicator), split = b ≥ 2 emulates b slices without NCCL (the blocked layout and slice arithmetic).
static int orth_blocks(const Ctx* c, int m, int64_t d, int impl) {
  if (impl != 2) return 0;                                 // the SIMT pass writes Z plain
  if (c->orth_split == 1) return 0;
  if (c->orth_split == -1) return (c->nccl_comm && d % (4 * c->world) == 0) ? c->world : 0;
  if (c->orth_split >= 2) return (c->world == 1 && d % (4 * c->orth_split) == 0) ? c->orth_split : 0;
  const bool big = (double)d * m * m >= (double)(1 << 28);     // C5: 2^30; C3, C4: ≤ 2^24 (NCCL latency wins there)
  return (c->world > 1 && c->nccl_comm && big && d % (4 * c->world) == 0) ? c->world : 0;
}

__global__ void add_into_f64_kernel(double* __restrict__ acc, const double* __restrict__ v, int64_t count) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < count) acc[e] += v[e];
}

// W[i][g·ds + x] = Wb[(g·m + i)·ds + x]
__global__ void unblock_kernel(const float* __restrict__ Wb, int m, int64_t ds, int blocks, float* __restrict__ W) {
  const int64_t d = ds * blocks;
  const int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (e >= (int64_t)m * d) return;
  const int64_t i = e / d, col = e % d, g = col / ds, x = col % ds;   // ds % 4 == 0: a float4 stays in one block
  *reinterpret_cast<float4*>(W + e) = *reinterpret_cast<const float4*>(Wb + (g * m + i) * ds + x);
}

// the exchange of the distributed mode: reduce-scatter of the d-blocked Z + all-reduce of S, one group
static ppca_status exchange_dist(Ctx* c, const float* Zb, float* Zg, size_t slice, double* S, size_t ns) {
  ncclResult_t r = g_nccl.GroupStart();
  if (r == ncclSuccess)
    r = g_nccl.ReduceScatter(Zb, Zg, slice, ncclFloat32, ncclSum, (ncclComm_t)c->nccl_comm, c->stream);
  if (r == ncclSuccess && ns) r = g_nccl.AllReduce(S, S, ns, ncclFloat64, ncclSum, (ncclComm_t)c->nccl_comm, c->stream);
  ncclResult_t r2 = g_nccl.GroupEnd();
  if (r != ncclSuccess || r2 != ncclSuccess)
    return set_error(c, PPCA_ERR_NCCL, "reduce-scatter Z / all-reduce S: %s", g_nccl.GetErrorString(r != ncclSuccess ? r : r2));
  c->collectives++;
  return PPCA_OK;
}

// W ← orth(Z) from the d-blocked Z (after exchange_dist when NCCL runs it).  One CholQR pass, fp64 Gram / factor /
// apply as in cholqr(); the Gram is the sum of the slice Grams (a fixed order: slices 0..G-1 in the emulation,
// NCCL's reduction order across ranks).
static ppca_status cholqr_dist(Ctx* c, float* Zb, const float* Zg, float* W, int m, int64_t d, int blocks) {
  const int64_t ds = d / blocks;
  const bool nccl = c->orth_split <= 0;                    // the real path (NCCL); otherwise the emulation
  double* G = (double*)scratch(c, S_GRAM, (size_t)2 * m * m * sizeof(double));
  double* Linv = (double*)scratch(c, S_SMALL, (size_t)m * m * sizeof(double) + 2 * m * sizeof(int) + 64);
  float* Wb = (float*)scratch(c, S_W2, (size_t)m * d * sizeof(float));
  float* Wg = (float*)scratch(c, S_DIST, (size_t)2 * m * ds * sizeof(float)) + (size_t)m * ds;
  if (!G || !Linv || !Wb || !Wg) return set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
  int* row_map = (int*)(Linv + (size_t)m * m);
  int* m_out = row_map + m;
  if (nccl) {
    PPCA_TRY(vec_gram(c, Zg, m, ds, G));
    PPCA_TRY(allreduce(c, G, (size_t)m * m, true));
  } else {
    for (int g = 0; g < blocks; ++g) {
      PPCA_TRY(vec_gram(c, Zb + (size_t)g * m * ds, m, ds, g ? G + (size_t)m * m : G));
      if (g) {
        add_into_f64_kernel<<<(unsigned)ceil_div((int64_t)m * m, 256), 256, 0, c->stream>>>(G, G + (size_t)m * m, (int64_t)m * m);
        PPCA_LAUNCH_CHECK(c, "add_into_f64");
      }
    }
  }
  PPCA_TRY(chol_inv_on(c, G, m, Linv, row_map, m_out, c->stream));
  if (nccl) {
    PPCA_TRY(apply_lower_on(c, Linv, m, Zg, ds, Wg, c->stream));
    ncclResult_t r = g_nccl.AllGather(Wg, Wb, (size_t)m * ds, ncclFloat32, (ncclComm_t)c->nccl_comm, c->stream);
    if (r != ncclSuccess) return set_error(c, PPCA_ERR_NCCL, "all-gather W: %s", g_nccl.GetErrorString(r));
    c->collectives++;
  } else {
    for (int g = 0; g < blocks; ++g)
      PPCA_TRY(apply_lower_on(c, Linv, m, Zb + (size_t)g * m * ds, ds, Wb + (size_t)g * m * ds, c->stream));
  }
  unblock_kernel<<<(unsigned)ceil_div((int64_t)m * d, 1024), 256, 0, c->stream>>>(Wb, m, ds, blocks, W);
  PPCA_LAUNCH_CHECK(c, "unblock");
  return PPCA_OK;
}

// ----------------------------------------------------------------------------- validation
static ppca_status check_matrix(Ctx* c, const ppca_matrix* X, int m) {
  if (!X || (!X->data && X->n_local > 0)) return set_error(c, PPCA_ERR_INVALID_ARG, "null matrix");
  if (X->d < 1 || X->ld < X->d || X->n_local < 0 || X->n_global < X->n_local)
    return set_error(c, PPCA_ERR_DIM_MISMATCH, "bad matrix dims n_local=%lld d=%lld ld=%lld", (long long)X->n_local,
                     (long long)X->d, (long long)X->ld);
  if (X->dtype != PPCA_F32 && X->dtype != PPCA_BF16 && X->dtype != PPCA_F32_SPLIT)
    return set_error(c, PPCA_ERR_INVALID_ARG, "bad dtype");
  if (X->dtype == PPCA_F32_SPLIT && (X->d % 8 || (reinterpret_cast<uintptr_t>(X->data) % 16)))
    return set_error(c, PPCA_ERR_INVALID_ARG, "PPCA_F32_SPLIT needs d %% 8 == 0 and a 16-byte aligned X");
  if ((X->ld * (int64_t)elt_size(X->dtype)) % 16) return set_error(c, PPCA_ERR_INVALID_ARG, "ld*elt %% 16 != 0");
  // the descriptor must describe exactly this rank's shard: kernels take row offsets from n_global
  if (c->world == 1 && X->n_global != X->n_local)
    return set_error(c, PPCA_ERR_DIM_MISMATCH, "one rank: n_global (%lld) must equal n_local (%lld)",
                     (long long)X->n_global, (long long)X->n_local);
  if (c->world > 1) {
    int64_t want;
    if (X->layout == PPCA_LAYOUT_INTERLEAVED) {
      const int64_t b = X->block_rows;
      if (b < 1 || b % c->world || (X->n_global % b) % c->world)
        return set_error(c, PPCA_ERR_INVALID_ARG, "INTERLEAVED: world must divide block_rows and the last block");
      want = (X->n_global / b) * (b / c->world) + (X->n_global % b) / c->world;
    } else {
      const int64_t per = ceil_div(X->n_global, (int64_t)c->world);
      want = std::max<int64_t>(0, std::min<int64_t>(per, X->n_global - (int64_t)c->rank * per));
    }
    if (X->n_local != want)
      return set_error(c, PPCA_ERR_DIM_MISMATCH, "rank %d: n_local = %lld, but the layout gives %lld rows", c->rank,
                       (long long)X->n_local, (long long)want);
  }
  if (m < 1) return set_error(c, PPCA_ERR_INVALID_ARG, "m must be >= 1");
  if (m > PPCA_MAX_M || m > X->d)
    return set_error(c, PPCA_ERR_TOO_MANY_COMPONENTS, "m=%d exceeds d=%lld or %d", m, (long long)X->d, PPCA_MAX_M);
  return PPCA_OK;
}

// local row range of global minibatch block s (reading R10)
static void block_range(const ppca_matrix* X, int world, int64_t b, int64_t s, int64_t* r0, int64_t* rows) {
  int64_t n = X->n_global, nb = ceil_div(n, b), nbf = n / b;
  s %= nb;
  int64_t q = b / world;
  if (s < nbf) {
    *r0 = s * q;
    *rows = q;
  } else {
    *r0 = nbf * q;
    *rows = (n - nbf * b) / world;
  }
}

}  // namespace ppca

using namespace ppca;

// ============================================================================= ABI
extern "C" {

const char* ppca_status_string(ppca_status s) {
  switch (s) {
    case PPCA_OK: return "ok";
    case PPCA_ERR_INVALID_ARG: return "invalid argument";
    case PPCA_ERR_DIM_MISMATCH: return "dimension mismatch";
    case PPCA_ERR_TOO_MANY_COMPONENTS: return "too many components";
    case PPCA_ERR_NONFINITE: return "non-finite update";
    case PPCA_ERR_DEGENERATE: return "degenerate denominator";
    case PPCA_ERR_SUBSPACE_COLLAPSE: return "subspace collapse";
    case PPCA_ERR_NO_CONVERGENCE: return "no convergence";
    case PPCA_ERR_CUDA: return "CUDA error";
    case PPCA_ERR_NCCL: return "NCCL error";
    case PPCA_ERR_UNSUPPORTED: return "unsupported";
  }
  return "unknown status";
}

int ppca_abi_version(void) { return PPCA_ABI_VERSION; }

ppca_status ppca_get_unique_id(void* uid_out) {
  if (!uid_out) return PPCA_ERR_INVALID_ARG;
  if (!nccl_load()) return PPCA_ERR_UNSUPPORTED;
  ncclUniqueId id;
  if (g_nccl.GetUniqueId(&id) != ncclSuccess) return PPCA_ERR_NCCL;
  memcpy(uid_out, &id, sizeof(id));
  return PPCA_OK;
}

ppca_status ppca_ctx_create(int device, void* stream, const void* uid, int rank, int world, ppca_ctx** out) {
  if (!out || world < 1 || rank < 0 || rank >= world) return PPCA_ERR_INVALID_ARG;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    cudaGetLastError();
    return PPCA_ERR_CUDA;
  }
  if (cudaSetDevice(device) != cudaSuccess) return PPCA_ERR_CUDA;
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, device);
  if (prop.major != 10) return PPCA_ERR_UNSUPPORTED;   // sm_100a build
  ppca_ctx* h = new ppca_ctx();
  Ctx* c = &h->c;
  c->device = device;
  c->rank = rank;
  c->world = world;
  c->sm_count = prop.multiProcessorCount;
  c->user_stream = (cudaStream_t)stream;
  c->stream = c->user_stream;
  // the library's own stream at the highest priority, the side stream (off-critical-path Ritz solves and
  // operand Grams) at the lowest: when both have CTAs waiting, the critical path's are dispatched first.
  // Every call orders the library stream after the caller's (enter()) and returns once its work is done.
  int prio_lo = 0, prio_hi = 0;
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  static const int use_prio = tune_env("PPCA_PRIO", 1);
  if (use_prio && prio_hi != prio_lo) {
    if (cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, prio_hi) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->fork_ev, cudaEventDisableTiming) != cudaSuccess) {
      delete h;
      return PPCA_ERR_CUDA;
    }
    c->own_stream = true;
  }
  if (cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, prio_lo) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_a, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_b, cudaEventDisableTiming) != cudaSuccess ||
      cudaMalloc(&c->d_err, sizeof(int)) != cudaSuccess || cudaMemset(c->d_err, 0, sizeof(int)) != cudaSuccess) {
    delete h;
    return PPCA_ERR_CUDA;
  }
  // world > 1 needs the NCCL unique id; world == 1 with an id creates a one-rank communicator, so every
  // collective call site of the path runs (and is tested) on a single GPU as well
  if (world > 1 && !uid) { delete h; return PPCA_ERR_INVALID_ARG; }
  if (uid) {
    if (!nccl_load()) { delete h; return PPCA_ERR_UNSUPPORTED; }
    ncclUniqueId id;
    memcpy(&id, uid, sizeof(id));
    ncclComm_t comm;
    if (g_nccl.CommInitRank(&comm, world, id, rank) != ncclSuccess) { delete h; return PPCA_ERR_NCCL; }
    int cnt = 0;
    if (g_nccl.CommCount && (g_nccl.CommCount(comm, &cnt) != ncclSuccess || cnt != world)) {
      g_nccl.CommDestroy(comm);
      delete h;
      return PPCA_ERR_NCCL;
    }
    c->nccl_comm = comm;
    if (rank == 0 && world > 1) fprintf(stderr, "[ppca] NCCL communicator: %d ranks (rank 0 on device %d)\n", world, device);
  }
  *out = h;
  return PPCA_OK;
}

ppca_status ppca_ctx_destroy(ppca_ctx* h) {
  if (!h) return PPCA_ERR_INVALID_ARG;
  Ctx* c = &h->c;
  enter(c);
  cudaStreamSynchronize(c->stream);
  if (c->side) cudaStreamSynchronize(c->side);
  for (int i = 0; i < Ctx::kSlots; ++i)
    if (c->slot_ptr[i]) cudaFree(c->slot_ptr[i]);
  if (c->d_err) cudaFree(c->d_err);
  if (c->flags) cudaFree(c->flags);
  if (c->ev_a) cudaEventDestroy(c->ev_a);
  if (c->ev_b) cudaEventDestroy(c->ev_b);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->own_stream) cudaStreamDestroy(c->stream);
  if (c->fork_ev) cudaEventDestroy(c->fork_ev);
  if (c->nccl_comm) g_nccl.CommDestroy((ncclComm_t)c->nccl_comm);
  pass_release(c);
  delete h;
  return PPCA_OK;
}

ppca_status ppca_last_error(const ppca_ctx* h, char* msg, size_t cap) {
  if (!h || !msg || cap == 0) return PPCA_ERR_INVALID_ARG;
  snprintf(msg, cap, "%s", h->c.last_error.c_str());
  return PPCA_OK;
}

int64_t ppca_launch_count(const ppca_ctx* h) { return h ? h->c.launches : -1; }
int64_t ppca_collective_count(const ppca_ctx* h) { return h ? h->c.collectives : -1; }

ppca_status ppca_set_orth_split(ppca_ctx* h, int split) {
  if (!h || split < -1 || split > 64) return PPCA_ERR_INVALID_ARG;
  h->c.orth_split = split;
  return PPCA_OK;
}

int ppca_experiments_enabled(void) {
#ifdef PPCA_EXPERIMENTS
  return 1;
#else
  return 0;
#endif
}

ppca_status ppca_set_timing(ppca_ctx* h, int enable) {
  if (!h) return PPCA_ERR_INVALID_ARG;
  h->c.timing = enable != 0;
  h->c.tev_used = 0;
  h->c.kev_used[0] = h->c.kev_used[1] = 0;
  return PPCA_OK;
}

ppca_status ppca_get_pass_time(ppca_ctx* h, double* ms_total, int64_t* passes) {
  if (!h || !ms_total || !passes) return PPCA_ERR_INVALID_ARG;
  enter(&h->c);
  return pass_time_collect(&h->c, ms_total, passes);
}

ppca_status ppca_get_kernel_time(ppca_ctx* h, int which, double* ms_total, int64_t* launches) {
  if (!h || !ms_total || !launches || which < 0 || which > 1) return PPCA_ERR_INVALID_ARG;
  enter(&h->c);
  return kernel_time_collect(&h->c, which, ms_total, launches);
}

// (undocumented, profiling) per-role mbarrier wait cycles of the tensor-core kernel A since last call
ppca_status ppca_debug_wait_counters(unsigned long long* out16) { return ppca::debug_wait_counters(out16); }

int ppca_last_pass_impl(const ppca_ctx* h) { return h ? h->c.last_impl : -1; }

int ppca_last_power_kernel(const ppca_ctx* h) { return h ? h->c.last_power_kernel : -1; }

ppca_status ppca_set_pass_impl(ppca_ctx* h, int impl) {
  if (!h || impl < 0 || impl > 4) return PPCA_ERR_INVALID_ARG;
  h->c.pass_impl = impl;
  return PPCA_OK;
}

ppca_status ppca_generate(ppca_ctx* h, const ppca_gen_spec* spec, void* X, int64_t ld, int64_t* n_local_out,
                          double* col_mean_host) {
  if (!h) return PPCA_ERR_INVALID_ARG;
  Ctx* c = &h->c;
  enter(c);
  PPCA_TRY(generate(c, spec, X, ld, n_local_out, col_mean_host));
  return finish(c, "ppca_generate");
}

ppca_status ppca_split_f32(ppca_ctx* h, void* X, int64_t n_local, int64_t d, int64_t ld) {
  if (!h) return PPCA_ERR_INVALID_ARG;
  Ctx* c = &h->c;
  enter(c);
  PPCA_TRY(split_f32(c, X, n_local, d, ld));
  return finish(c, "ppca_split_f32");
}

ppca_status ppca_upload_rows(ppca_ctx* h, const void* host, int64_t rows, int64_t ld_host, const ppca_matrix* X,
                             int64_t r0) {
  if (!h || !X || (!host && rows > 0)) return PPCA_ERR_INVALID_ARG;
  Ctx* c = &h->c;
  enter(c);
  if (rows < 0 || r0 < 0 || r0 + rows > X->n_local || ld_host < X->d || X->ld < X->d)
    return set_error(c, PPCA_ERR_INVALID_ARG, "upload rows [%lld, %lld) outside the shard of %lld rows",
                     (long long)r0, (long long)(r0 + rows), (long long)X->n_local);
  if (rows == 0) return PPCA_OK;
  const size_t elt = X->dtype == PPCA_BF16 ? 2 : 4;          // logical element (the split planes are 4 B)
  uint8_t* dst = static_cast<uint8_t*>(const_cast<void*>(X->data)) + (size_t)r0 * X->ld * elt;
  PPCA_TRY(check_cuda(c, cudaMemcpy2DAsync(dst, (size_t)X->ld * elt, host, (size_t)ld_host * elt, (size_t)X->d * elt,
                                           (size_t)rows, cudaMemcpyHostToDevice, c->stream), "upload rows"));
  if (X->dtype == PPCA_F32_SPLIT) PPCA_TRY(split_f32(c, dst, rows, X->d, X->ld));
  return finish(c, "ppca_upload_rows");
}

ppca_status ppca_philox_words(ppca_ctx* h, uint64_t seed, uint32_t stream, uint64_t first, int64_t count,
                              uint32_t* out) {
  if (!h || (!out && count > 0)) return PPCA_ERR_INVALID_ARG;
  Ctx* c = &h->c;
  enter(c);
  PPCA_TRY(philox_words(c, seed, stream, first, count, out));
  return finish(c, "ppca_philox_words");
}

// ---------------------------------------------------------------------------- power priming
ppca_status ppca_prime_power(ppca_ctx* h, const ppca_matrix* X, int m, int iters, double eps, uint64_t init_seed,
                             float* W, double* theta_hist_host, int* iters_done) {
  if (!h) return PPCA_ERR_INVALID_ARG;
  Ctx* c = &h->c;
  enter(c);
  if (iters_done) *iters_done = 0;
  PPCA_TRY(check_matrix(c, X, m));
  if (!W || iters < 0 || !(eps == eps)) return set_error(c, PPCA_ERR_INVALID_ARG, "null W, iters < 0 or NaN eps");
  const bool stop_rule = eps > 0.0;
  const int64_t d = X->d;
  // all scratch up front (no reallocation while the side stream is busy)
  float* Z = (float*)scratch(c, S_Z, (size_t)m * d * sizeof(float));
  if (init_seed) {
    // W_0 = Q-factor of a Gaussian block: one fp64 CholQR pass is exact to ε64·κ² (κ of an m×d Gaussian block
    // ≈ (√d + √m)/(√d − √m), below 2 for the workloads), so the second pass of CholQR2 would change nothing
    if (!Z) return set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
    PPCA_TRY(init_rows(c, init_seed, Z, m, d));
    PPCA_TRY(cholqr(c, Z, W, m, d, 0.0, nullptr, (double)m * 4 <= (double)d ? 1 : 2));
  }
  double* Sbuf = (double*)scratch(c, S_S, (size_t)4 * m * m * sizeof(double));      // S[2], Bm[2]
  double* theta_dev = (double*)scratch(c, S_TC2, (size_t)std::max(1, iters) * m * sizeof(double) + (size_t)m * m * sizeof(double));
  if (!Z || !Sbuf || !theta_dev) return set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
  float* Wold = stop_rule ? (float*)scratch(c, S_EPS, (size_t)m * d * sizeof(float) + (size_t)m * sizeof(double)) : nullptr;
  if (stop_rule && !Wold) return set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
  double* dots = stop_rule ? reinterpret_cast<double*>(Wold + (size_t)m * d) : nullptr;
  std::vector<double> hdots(stop_rule ? m : 0);
  int done = 0;
  if (theta_hist_host && iters > 0)
    PPCA_TRY(check_cuda(c, cudaMemsetAsync(theta_dev, 0, (size_t)iters * m * sizeof(double), c->stream), "zero theta"));
  PassPlan plan;
  PPCA_TRY(pass_prepare(c, X, m, &plan));
  const int oblk = orth_blocks(c, m, d, plan.impl);        // > 0: the distributed CholQR (§6)
  float* Zg = nullptr;
  if (oblk > 0) {
    Zg = (float*)scratch(c, S_DIST, (size_t)2 * m * (d / oblk) * sizeof(float));
    if (!Zg) return set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
  }
  // pre-touch the scratch the loop uses so no allocation happens while the side stream is busy
  if (!scratch(c, S_EVAL, (size_t)3 * m * m * sizeof(double)) || !scratch(c, S_GRAM, (size_t)2 * m * m * sizeof(double)) ||
      !scratch(c, S_SMALL, (size_t)m * m * sizeof(double) + 2 * m * sizeof(int) + 64) ||
      !scratch(c, S_W2, (size_t)m * d * sizeof(float)) || !scratch(c, S_SIDE_PART, vec_gram_part_bytes(c, m, d)) ||
      !scratch(c, S_ZGRAM, zgram_part_bytes(m, d)))
    return set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
  // the next pass operand W' written by CholQR's apply (small d·m, one rank's replicated CholQR): two buffers —
  // the apply of iteration t writes wp_buf[t & 1] while the side Gram of iteration t may still read the other
  const int mp_op = (m + 15) & ~15;
  const bool fuse_prep = plan.impl == 2 && oblk == 0 && wprep_fusable(c, m, mp_op, d);
  const size_t wp_bytes = (size_t)2 * mp_op * d * 2 + (size_t)m * d * 4 + 256;
  uint8_t* wp_buf[2] = {nullptr, nullptr};
  if (fuse_prep) {
    wp_buf[0] = (uint8_t*)scratch(c, S_WPREP, wp_bytes);
    wp_buf[1] = (uint8_t*)scratch(c, S_TC1, wp_bytes);   // prep_w's own buffer (pass 0)
    if (!wp_buf[0] || !wp_buf[1]) return set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
  }
  c->wprep_for = nullptr;
  cudaEvent_t ev_main[2], ev_side[2], ev_prep, ev_gram;
  cudaEventCreateWithFlags(&ev_prep, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&ev_gram, cudaEventDisableTiming);
  cudaEventRecord(ev_gram, c->side);
  for (int i = 0; i < 2; ++i) {
    cudaEventCreateWithFlags(&ev_main[i], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ev_side[i], cudaEventDisableTiming);
    cudaEventRecord(ev_side[i], c->side);
  }
  ppca_status st = PPCA_OK;
  c->side_busy = theta_hist_host != nullptr;
  // one GPU with the θ history: S only feeds the side-stream Ritz solve, so its reduction moves there too
  c->s_defer = theta_hist_host != nullptr && c->nccl_comm == nullptr;
  // no θ history on one rank: S = YᵀY of the pass is not used at all (W comes from Z alone)
  c->s_skip = theta_hist_host == nullptr && c->nccl_comm == nullptr;
  if (c->s_defer) {
    cudaEventCreateWithFlags(&c->s_ev_pass, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&c->s_ev_red, cudaEventDisableTiming);
    cudaEventRecord(c->s_ev_red, c->side);
  }
  for (int t = 0; t < iters && st == PPCA_OK; ++t) {
    double* S = Sbuf + (size_t)(t & 1) * m * m;
    double* Bm = Sbuf + (size_t)(2 + (t & 1)) * m * m;
    if (theta_hist_host) {
      cudaStreamWaitEvent(c->stream, ev_side[t & 1], 0);   // Ritz t-2 done with S, Bm
      cudaStreamWaitEvent(c->stream, ev_gram, 0);          // the side Gram of W'_{t-1} read it before prep_w rewrites
    }
    c->z_block_cols = oblk > 0 ? d / oblk : 0;               // the pass writes Z d-blocked for the slices
    // one rank, replicated CholQR: the pass's Z reduction may also leave the CholQR's Gram ZᵀZ
    c->zgram_want = oblk == 0 && c->nccl_comm == nullptr;
    c->zgram_done = false;
    st = pass_power(c, X, &plan, W, m, Z, S);               // Z = YᵀX, S = YᵀY  (local)
    const bool gram_ready = c->zgram_done;
    c->zgram_want = c->zgram_done = false;
    c->z_block_cols = 0;
    if (st != PPCA_OK) break;
    if (theta_hist_host) {
      // side stream, once the pass is done (a Gram overlapping the persistent pass would take its SMs): Bm =
      // W'W'ᵀ of the operand the pass used — concurrent with the main stream's CholQR — then the pPCA-for-free
      // Ritz values of span(W'_t) once S_t is reduced
      cudaEventRecord(ev_prep, c->stream);
      cudaStreamWaitEvent(c->side, ev_prep, 0);
      st = vec_gram_on(c, plan.Wop, m, d, Bm, c->side, S_SIDE_PART);
      if (st != PPCA_OK) break;
      cudaEventRecord(ev_gram, c->side);
      st = pass_reduce_deferred_s(c, S, c->side);
      if (st != PPCA_OK) break;
    }
    if (oblk > 0 && c->orth_split <= 0)
      st = exchange_dist(c, Z, Zg, (size_t)m * (d / oblk), S, (size_t)m * m);   // slices of Z + S, one group
    else if (oblk == 0)
      st = allreduce_zs(c, Z, (size_t)m * d, S, (size_t)m * m);   // the only collective: [Z | S], one group
    if (st != PPCA_OK) break;
    if (theta_hist_host) {
      cudaEventRecord(ev_main[t & 1], c->stream);
      cudaStreamWaitEvent(c->side, ev_main[t & 1], 0);
      st = ritz_solve(c, S, Bm, m, theta_dev + (size_t)t * m, nullptr, c->side);   // values only
      cudaEventRecord(ev_side[t & 1], c->side);
      if (st != PPCA_OK) break;
    }
    // W ← orth(Z): one fp64 Cholesky-QR pass (κ(Z)² ε64 ≪ fp32 rounding for power iterates); it rewrites
    // W (the SIMT pass's operand: there the side Gram reads W itself, so wait for it) and the next prep_w
    // rewrites W' (the wait at the top of the loop)
    if (theta_hist_host && plan.impl != 2) cudaStreamWaitEvent(c->stream, ev_gram, 0);
    if (stop_rule) {
      st = check_cuda(c, cudaMemcpyAsync(Wold, W, (size_t)m * d * sizeof(float), cudaMemcpyDeviceToDevice, c->stream),
                      "keep W_t");
      if (st != PPCA_OK) break;
    }
    WPrep wp{};
    if (fuse_prep) {
      uint8_t* b = wp_buf[t & 1];
      wp.Wb = reinterpret_cast<__nv_bfloat16*>(b);
      wp.Wr = reinterpret_cast<float*>(b + (((size_t)2 * mp_op * d * 2 + 255) & ~(size_t)255));
      wp.lo_off = (int64_t)mp_op * d;
    }
    st = oblk > 0 ? cholqr_dist(c, Z, Zg, W, m, d, oblk)
                  : cholqr(c, Z, W, m, d, 0.0, nullptr, 1, gram_ready, fuse_prep ? &wp : nullptr);
    if (st != PPCA_OK) break;
    if (fuse_prep) {
      c->wprep_for = W;
      c->wprep_b = wp.Wb;
      c->wprep_r = wp.Wr;
    }
    done = t + 1;
    if (stop_rule) {                                 // P L61-62: stop once every column moved less than eps
      st = row_dots(c, W, Wold, m, d, dots);
      if (st == PPCA_OK)
        st = check_cuda(c, cudaMemcpyAsync(hdots.data(), dots, (size_t)m * sizeof(double), cudaMemcpyDeviceToHost,
                                           c->stream), "stop rule");
      if (st == PPCA_OK) st = check_cuda(c, cudaStreamSynchronize(c->stream), "stop rule");
      if (st != PPCA_OK) break;
      double worst = 0.0;                            // ‖w' − s·w‖² = 2 − 2|⟨w', w⟩| for unit columns
      for (int j = 0; j < m; ++j) worst = std::max(worst, std::sqrt(std::max(0.0, 2.0 - 2.0 * std::fabs(hdots[j]))));
      if (worst < eps) break;
    }
  }
  c->prep_ev = nullptr;
  c->wprep_for = nullptr;
  c->s_skip = false;
  c->side_busy = false;
  if (c->s_pending) pass_reduce_deferred_s(c, Sbuf, c->side);   // an aborted loop: drain (result unused)
  ppca_status st2 = finish(c, "ppca_prime_power");
  if (c->s_defer) {
    cudaEventDestroy(c->s_ev_pass);
    cudaEventDestroy(c->s_ev_red);
    c->s_ev_pass = c->s_ev_red = nullptr;
    c->s_defer = false;
  }
  for (int i = 0; i < 2; ++i) {
    cudaEventDestroy(ev_main[i]);
    cudaEventDestroy(ev_side[i]);
  }
  cudaEventDestroy(ev_prep);
  cudaEventDestroy(ev_gram);
  if (st != PPCA_OK) return st;
  if (st2 != PPCA_OK) return st2;
  if (theta_hist_host && iters > 0) {
    if (cudaMemcpy(theta_hist_host, theta_dev, (size_t)iters * m * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess)
      return set_error(c, PPCA_ERR_CUDA, "copy theta");
  }
  if (iters_done) *iters_done = done;
  return PPCA_OK;
}

// ---------------------------------------------------------------------------- minibatch primings
static ppca_status minibatch_common(Ctx* c, const ppca_matrix* X, int m, int batch, int64_t steps, uint64_t init_seed,
                                    float* W, float* vel, int64_t* step_io, bool eigengame, double alpha, double mu) {
  PPCA_TRY(check_matrix(c, X, m));
  if (!W || !vel || !step_io || steps < 0 || batch < 1) return set_error(c, PPCA_ERR_INVALID_ARG, "bad minibatch args");
  if (batch % c->world) return set_error(c, PPCA_ERR_INVALID_ARG, "world must divide batch");
  if (c->world > 1 && (X->layout != PPCA_LAYOUT_INTERLEAVED || X->block_rows != batch))
    return set_error(c, PPCA_ERR_INVALID_ARG, "minibatch priming on >1 GPU needs the INTERLEAVED layout with block_rows == batch");
  if (((X->n_global % batch) % c->world) != 0) return set_error(c, PPCA_ERR_INVALID_ARG, "world must divide the last block");
  const int64_t d = X->d;
  if (init_seed) {
    PPCA_TRY(init_rows(c, init_seed, W, m, d));
    PPCA_TRY(check_cuda(c, cudaMemsetAsync(vel, 0, (size_t)m * d * sizeof(float), c->stream), "zero velocity"));
  }
  float* Q = (float*)scratch(c, S_Z, (size_t)m * d * sizeof(float));
  double* P = (double*)scratch(c, S_S, (size_t)m * m * sizeof(double));
  if (!Q || !P) return set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
  int64_t s0 = *step_io;
  if (!eigengame) {
    // short windows on one GPU: every step inside one persistent kernel (the multi-launch step below is
    // launch-latency bound there)
    ppca_status pst;
    if (oja_persistent(c, X, m, batch, alpha, mu, s0, steps, W, vel, &pst)) {
      PPCA_TRY(pst);
      *step_io = s0 + steps;
      return PPCA_OK;
    }
  }
  const size_t row_bytes = (size_t)X->ld * elt_size(X->dtype);
  for (int64_t s = s0; s < s0 + steps; ++s) {
    int64_t r0, rows;
    block_range(X, c->world, batch, s, &r0, &rows);
    // the step's products Q = X_bᵀ(X_b Wᵀ), P = (X_b Wᵀ)ᵀ(X_b Wᵀ) are one streaming pass over the window:
    // the tensor-core pass (K-split across the SMs for a short window) when the window is large enough
    ppca_matrix Xw = *X;
    Xw.data = static_cast<const uint8_t*>(X->data) + (size_t)r0 * row_bytes;
    Xw.n_local = rows;
    PassPlan plan;
    if (pass_prepare(c, &Xw, m, &plan) != PPCA_OK) plan.impl = 1;   // e.g. a short last block
    plan.precise = true;
    if (X->dtype == PPCA_F32) plan.impl = 1;   // the converter kernels read X_hi only in product 2
    if (plan.impl == 2) {
      // one GPU, EigenGame: Z stays as the window pass's row-group partials, summed by the update kernel
      c->zp_pending = false;
      c->zp_defer = eigengame && !c->nccl_comm;
      const ppca_status pst = pass_power(c, &Xw, &plan, W, m, Q, P);
      c->zp_defer = false;
      c->wprep_for = nullptr;                       // adopted by the pass (or not wanted)
      PPCA_TRY(pst);
    } else {
      c->wprep_for = nullptr;
      float* Y = (float*)scratch(c, S_Y, (size_t)std::max<int64_t>(1, rows) * m * sizeof(float));
      if (!Y) return set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
      c->last_impl = 1;
      PPCA_TRY(xw(c, X, r0, rows, W, m, Y));
      PPCA_TRY(ytx(c, X, r0, rows, Y, m, Q));
      PPCA_TRY(yty(c, Y, m, rows, P));
    }
    PPCA_TRY(allreduce_zs(c, Q, (size_t)m * d, P, (size_t)m * m));
    if (eigengame) {
      // the next window pass's operand split written by the update kernel itself (m = padded m: no zero rows)
      WPrep wp{};
      static const bool eg_prep = tune_env("PPCA_EG_PREP", 1) != 0;
      bool want = eg_prep && plan.impl == 2 && ((m + 15) & ~15) == m && X->dtype != PPCA_F32;
      if (want) {
        const size_t bytes = (size_t)2 * m * d * 2 + (size_t)m * d * 4 + 256;
        uint8_t* b = (uint8_t*)scratch(c, S_TC1, bytes);   // prep_w's buffer; nothing else reads it until then
        want = b != nullptr;
        if (want) {
          wp.Wb = reinterpret_cast<__nv_bfloat16*>(b);
          wp.Wr = reinterpret_cast<float*>(b + (((size_t)2 * m * d * 2 + 255) & ~(size_t)255));
          wp.lo_off = (int64_t)m * d;
        }
      }
      bool done = false;
      PPCA_TRY(eigengame_update(c, Q, P, W, vel, m, d, alpha, mu, want ? &wp : nullptr, &done));
      if (done) {
        c->wprep_for = W;
        c->wprep_b = wp.Wb;
        c->wprep_r = wp.Wr;
      }
    } else {
      PPCA_TRY(pass_reduce_deferred_z(c, Q));
      PPCA_TRY(oja_update(c, Q, P, W, vel, m, d, alpha, mu));
    }
    c->zp_pending = false;
  }
  *step_io = s0 + steps;
  return PPCA_OK;
}

ppca_status ppca_prime_oja(ppca_ctx* h, const ppca_matrix* X, int m, int batch, double alpha, double momentum,
                           int64_t steps, uint64_t init_seed, float* W, float* velocity, int64_t* step_io) {
  if (!h) return PPCA_ERR_INVALID_ARG;
  Ctx* c = &h->c;
  enter(c);
  PPCA_TRY(minibatch_common(c, X, m, batch, steps, init_seed, W, velocity, step_io, false, alpha, momentum));
  return finish(c, "ppca_prime_oja");
}

ppca_status ppca_prime_eigengame(ppca_ctx* h, const ppca_matrix* X, int m, int batch, double alpha, double momentum,
                                 int64_t steps, uint64_t init_seed, float* V, float* velocity, int64_t* step_io) {
  if (!h) return PPCA_ERR_INVALID_ARG;
  Ctx* c = &h->c;
  enter(c);
  PPCA_TRY(minibatch_common(c, X, m, batch, steps, init_seed, V, velocity, step_io, true, alpha, momentum));
  return finish(c, "ppca_prime_eigengame");
}

// ---------------------------------------------------------------------------- refine
// Alg. 1 steps 2-5 (P L47-51).  sample_fraction ≥ 1: all rows; otherwise only the 128-row tiles whose
// Philox uniform (seed, stream 7, tile key) is < sample_fraction are projected (P L378 "we only project 10%
// of the data"; reading R25) and θ are rescaled by n_global / rows used.
static ppca_status refine_impl(Ctx* c, const ppca_matrix* X, const float* V, int m, int k, double fraction,
                               uint64_t sample_seed, float* E, double* theta_host, int* subspace_dim,
                               int64_t* rows_used, unsigned flags = 0) {
  PPCA_TRY(check_matrix(c, X, m));
  if (!V || !E || k < 1 || k > m) return set_error(c, PPCA_ERR_INVALID_ARG, "bad refine args (k=%d, m=%d)", k, m);
  if (!(fraction > 0.0)) return set_error(c, PPCA_ERR_INVALID_ARG, "sample fraction must be > 0");
  const int64_t d = X->d;
  float* B = (float*)scratch(c, S_W3, (size_t)m * d * sizeof(float));
  double* S = (double*)scratch(c, S_S, (size_t)2 * m * m * sizeof(double) + 16);
  double* out = (double*)scratch(c, S_TC2, (size_t)m * sizeof(double) + (size_t)m * m * sizeof(double));
  if (!B || !S || !out) return set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
  double* Bm = S + (size_t)m * m;
  double* theta_dev = out;
  double* R = out + m;
  // row-tile sample (host: the Philox of common.cuh; the list is tiny — n_local/128 entries)
  std::vector<int32_t> tiles;
  double rows_local = (double)X->n_local;
  const bool sampled = fraction < 1.0;
  if (sampled) {
    const int64_t tile = 128, nt = ceil_div(X->n_local, tile);
    const int64_t r0 = X->layout == PPCA_LAYOUT_CONTIGUOUS ? c->rank * ceil_div(X->n_global, (int64_t)c->world) : 0;
    rows_local = 0.0;
    for (int64_t t = 0; t < nt; ++t) {
      // key = the global index of the tile's first row (R25): distinct for every tile of every rank, so no two
      // tiles share a draw; INTERLEAVED shards key on (rank, local tile) in a disjoint range
      const uint64_t key = X->layout == PPCA_LAYOUT_CONTIGUOUS ? (uint64_t)(r0 + t * tile)
                                                               : (1ull << 62) + ((uint64_t)c->rank << 40) + (uint64_t)t;
      if (u32_to_unit(philox_word(sample_seed, 7, key)) < fraction) {
        tiles.push_back((int32_t)t);
        rows_local += (double)(std::min(X->n_local, (t + 1) * tile) - t * tile);
      }
    }
  }
  double rows_total = rows_local;
  if (c->nccl_comm) {
    double* cnt = S + 2 * (size_t)m * m;
    PPCA_TRY(check_cuda(c, cudaMemcpyAsync(cnt, &rows_local, sizeof(double), cudaMemcpyHostToDevice, c->stream), "count"));
    PPCA_TRY(allreduce(c, cnt, 1, true));
    PPCA_TRY(check_cuda(c, cudaMemcpyAsync(&rows_total, cnt, sizeof(double), cudaMemcpyDeviceToHost, c->stream), "count"));
    PPCA_TRY(check_cuda(c, cudaStreamSynchronize(c->stream), "count"));
  }
  if (sampled && rows_total <= 0.0) return set_error(c, PPCA_ERR_INVALID_ARG, "the row sample is empty");
  int mm = m;
  if (flags & PPCA_REFINE_ORTHONORMAL) {
    // the caller guarantees orthonormal rows (ppca_prime_power's W): B = V.  The Rayleigh–Ritz step is the
    // generalized one with the Gram of the operand rows, so θ and E are exact for span V regardless
    PPCA_TRY(check_cuda(c, cudaMemcpyAsync(B, V, (size_t)m * d * sizeof(float), cudaMemcpyDeviceToDevice, c->stream),
                        "copy V"));
  } else {
    PPCA_TRY(check_cuda(c, cudaMemcpyAsync(B, V, (size_t)m * d * sizeof(float), cudaMemcpyDeviceToDevice, c->stream),
                        "copy V"));
    PPCA_TRY(normalize_rows(c, B, m, d));                 // current_components
    // B = orth(V); a direction whose relative residual is < 1e-6 is dropped (SPEC L51 drops < 1e-10 in
    // fp64; fp32 inputs cannot resolve residuals below ~1e-7 — DESIGN.md reading R14)
    PPCA_TRY(cholqr2(c, B, m, d, 1e-6, &mm));
    if (mm < k) {
      finish(c, "ppca_refine");
      return set_error(c, PPCA_ERR_SUBSPACE_COLLAPSE, "only %d of %d directions survive", mm, k);
    }
  }
  PassPlan plan;
  PPCA_TRY(pass_prepare(c, X, mm, &plan));
  if (sampled) {
    int32_t* td = (int32_t*)scratch(c, S_TILES, std::max<size_t>(1, tiles.size()) * sizeof(int32_t));
    if (!td) return set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
    if (!tiles.empty())
      PPCA_TRY(check_cuda(c, cudaMemcpyAsync(td, tiles.data(), tiles.size() * sizeof(int32_t), cudaMemcpyHostToDevice,
                                             c->stream), "copy tiles"));
    plan.tiles_dev = td;
    plan.tiles_host = tiles.data();
    plan.ntiles_sel = (int64_t)tiles.size();
  }
  PPCA_TRY(pass_gram(c, X, &plan, B, mm, S));            // S = (XBᵀ)ᵀ(XBᵀ) over the (sampled) rows
  PPCA_TRY(allreduce(c, S, (size_t)mm * mm, true));
  const float* Bop = plan.Wop;                            // the operand rows the pass used
  PPCA_TRY(vec_gram(c, Bop, mm, d, Bm));
  PPCA_TRY(ritz_solve(c, S, Bm, mm, theta_dev, R, c->stream, k));   // the k largest pairs only
  PPCA_TRY(lift_rows(c, R, mm, Bop, mm, k, d, E, true, c->stream));
  PPCA_TRY(finish(c, "ppca_refine"));
  if (theta_host) {
    if (cudaMemcpy(theta_host, theta_dev, (size_t)k * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess)
      return set_error(c, PPCA_ERR_CUDA, "copy theta");
    if (sampled)
      for (int i = 0; i < k; ++i) theta_host[i] *= (double)X->n_global / rows_total;
  }
  if (subspace_dim) *subspace_dim = mm;
  if (rows_used) *rows_used = (int64_t)rows_total;
  return PPCA_OK;
}

ppca_status ppca_refine(ppca_ctx* h, const ppca_matrix* X, const float* V, int m, int k, float* E, double* theta_host,
                        int* subspace_dim) {
  if (!h) return PPCA_ERR_INVALID_ARG;
  enter(&h->c);
  return refine_impl(&h->c, X, V, m, k, 1.0, 0, E, theta_host, subspace_dim, nullptr);
}

ppca_status ppca_refine_ex(ppca_ctx* h, const ppca_matrix* X, const float* V, int m, int k, unsigned flags, float* E,
                           double* theta_host, int* subspace_dim) {
  if (!h) return PPCA_ERR_INVALID_ARG;
  if (flags & ~(unsigned)PPCA_REFINE_ORTHONORMAL) return set_error(&h->c, PPCA_ERR_INVALID_ARG, "unknown refine flags");
  enter(&h->c);
  return refine_impl(&h->c, X, V, m, k, 1.0, 0, E, theta_host, subspace_dim, nullptr, flags);
}

ppca_status ppca_refine_sampled(ppca_ctx* h, const ppca_matrix* X, const float* V, int m, int k, double fraction,
                                uint64_t sample_seed, float* E, double* theta_host, int* subspace_dim,
                                int64_t* rows_used) {
  if (!h) return PPCA_ERR_INVALID_ARG;
  enter(&h->c);
  return refine_impl(&h->c, X, V, m, k, fraction, sample_seed, E, theta_host, subspace_dim, rows_used);
}

// ---------------------------------------------------------------------------- Prop. 3 checker (NEXT-4)
// PAPER.md §4.2 Prop. 3 (L293-302), reading R28: B = orth(V) as the refine builds it, S = the
// projected Gram of the pass, G = the Gram of the stacked [B_op; T] (one vector-Gram launch gives BBᵀ — the
// metric of the operand rows — and the coordinates B t_i together), then prop3_device.
ppca_status ppca_check_prop3(ppca_ctx* h, const ppca_matrix* X, const float* V, int m, const float* T, int upto,
                             double tol, double* angles_host, int* flags_host) {
  if (!h) return PPCA_ERR_INVALID_ARG;
  Ctx* c = &h->c;
  enter(c);
  PPCA_TRY(check_matrix(c, X, m));
  if (!V || !T || !angles_host || !flags_host || upto < 1 || upto > PPCA_MAX_M || !(tol >= 0.0))
    return set_error(c, PPCA_ERR_INVALID_ARG, "bad check_prop3 args (upto=%d)", upto);
  const int64_t d = X->d;
  float* B = (float*)scratch(c, S_W3, (size_t)m * d * sizeof(float));
  double* S = (double*)scratch(c, S_S, (size_t)2 * m * m * sizeof(double) + 16);
  if (!B || !S) return set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
  PPCA_TRY(check_cuda(c, cudaMemcpyAsync(B, V, (size_t)m * d * sizeof(float), cudaMemcpyDeviceToDevice, c->stream), "copy V"));
  PPCA_TRY(normalize_rows(c, B, m, d));
  int mm = m;
  PPCA_TRY(cholqr2(c, B, m, d, 1e-6, &mm));               // the refine's orth(V) (reading R14)
  if (mm < upto) {
    finish(c, "ppca_check_prop3");
    return set_error(c, PPCA_ERR_SUBSPACE_COLLAPSE, "span V has dimension %d < upto = %d", mm, upto);
  }
  PassPlan plan;
  PPCA_TRY(pass_prepare(c, X, mm, &plan));
  PPCA_TRY(pass_gram(c, X, &plan, B, mm, S));
  PPCA_TRY(allreduce(c, S, (size_t)mm * mm, true));
  const int g = mm + upto;
  float* stack = (float*)scratch(c, S_P3F, (size_t)g * d * sizeof(float));
  double* G = (double*)scratch(c, S_GRAM, (size_t)g * g * sizeof(double));
  if (!stack || !G) return set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
  PPCA_TRY(check_cuda(c, cudaMemcpyAsync(stack, plan.Wop, (size_t)mm * d * sizeof(float), cudaMemcpyDeviceToDevice,
                                         c->stream), "stack B"));
  PPCA_TRY(check_cuda(c, cudaMemcpyAsync(stack + (size_t)mm * d, T, (size_t)upto * d * sizeof(float),
                                         cudaMemcpyDeviceToDevice, c->stream), "stack T"));
  PPCA_TRY(vec_gram(c, stack, g, d, G));
  std::vector<double> ratio(upto);
  PPCA_TRY(prop3_device(c, G, g, S, mm, upto, ratio.data(), angles_host));
  PPCA_TRY(finish(c, "ppca_check_prop3"));
  bool chain = true;                                       // flag i: conditions 1 … i all hold (R28)
  for (int i = 0; i < upto; ++i) {
    chain = chain && angles_host[i] <= tol;
    flags_host[i] = chain ? 1 : 0;
  }
  return PPCA_OK;
}

// ---------------------------------------------------------------------------- Theorem 1 assertion (NEXT-4)
// P L308-312 with Prop. 3 (L293-302): upto = the leading run of Prop. 3 conditions that hold; on it pPCA's i-th
// vector is π_S(e_i)/‖π_S(e_i)‖, the vector of S closest to e_i, so ∠(pPCA_i, e_i) ≤ ∠(v_i, e_i) (+ tol).
ppca_status ppca_check_theorem1(ppca_ctx* h, const ppca_matrix* X, const float* V, int m, int k, const float* T,
                                double tol, int* upto_out, double* ang_priming_host, double* ang_ppca_host,
                                int* holds_out) {
  if (!h) return PPCA_ERR_INVALID_ARG;
  Ctx* c = &h->c;
  enter(c);
  if (!V || !T || !upto_out || !ang_priming_host || !ang_ppca_host || !holds_out || k < 1 || k > m || !(tol >= 0.0))
    return set_error(c, PPCA_ERR_INVALID_ARG, "bad check_theorem1 args (k=%d, m=%d)", k, m);
  std::vector<double> cang(k);
  std::vector<int> flags(k);
  PPCA_TRY(ppca_check_prop3(h, X, V, m, T, k, tol, cang.data(), flags.data()));
  int upto = 0;
  while (upto < k && flags[upto]) ++upto;
  const int64_t d = X->d;
  float* buf = (float*)scratch(c, S_P3F, (size_t)2 * k * d * sizeof(float));
  double* dots = (double*)scratch(c, S_ROWRED, (size_t)2 * std::max(k, PPCA_MAX_M) * sizeof(double));
  if (!buf || !dots) return set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
  float* E = buf;
  float* Vn = buf + (size_t)k * d;
  std::vector<double> th(k);
  int dim = 0;
  PPCA_TRY(refine_impl(c, X, V, m, k, 1.0, 0, E, th.data(), &dim, nullptr));
  PPCA_TRY(check_cuda(c, cudaMemcpyAsync(Vn, V, (size_t)k * d * sizeof(float), cudaMemcpyDeviceToDevice, c->stream),
                      "copy V"));
  PPCA_TRY(normalize_rows(c, Vn, k, d));                  // e_i^PRIMING = v_i / ‖v_i‖
  PPCA_TRY(row_dots(c, Vn, T, k, d, dots));
  PPCA_TRY(row_dots(c, E, T, k, d, dots + k));
  PPCA_TRY(finish(c, "ppca_check_theorem1"));
  std::vector<double> hd(2 * k);
  if (cudaMemcpy(hd.data(), dots, 2 * k * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess)
    return set_error(c, PPCA_ERR_CUDA, "copy dots");
  int holds = 1;
  for (int i = 0; i < k; ++i) {
    ang_priming_host[i] = acos(std::min(1.0, fabs(hd[i])));
    ang_ppca_host[i] = acos(std::min(1.0, fabs(hd[k + i])));
    if (i < upto && ang_ppca_host[i] > ang_priming_host[i] + tol) holds = 0;
  }
  *upto_out = upto;
  *holds_out = holds;
  return PPCA_OK;
}

// ---------------------------------------------------------------------------- eval / support
ppca_status ppca_eval(ppca_ctx* h, const float* E, const float* T, int k, int64_t d, const double* thr_host, int nthr,
                      double* angles_host, int* lces_host) {
  if (!h) return PPCA_ERR_INVALID_ARG;
  Ctx* c = &h->c;
  enter(c);
  if (!E || !T || k < 1 || d < 1 || (nthr > 0 && (!thr_host || !lces_host)))
    return set_error(c, PPCA_ERR_INVALID_ARG, "bad eval args");
  double* dots = (double*)scratch(c, S_ROWRED, (size_t)std::max(k, PPCA_MAX_M) * sizeof(double));
  PPCA_TRY(row_dots(c, E, T, k, d, dots));
  PPCA_TRY(finish(c, "ppca_eval"));
  std::vector<double> hd(k), ang(k);
  if (cudaMemcpy(hd.data(), dots, k * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess)
    return set_error(c, PPCA_ERR_CUDA, "copy dots");
  for (int i = 0; i < k; ++i) ang[i] = acos(std::min(1.0, fabs(hd[i])));
  if (angles_host) memcpy(angles_host, ang.data(), k * sizeof(double));
  for (int t = 0; t < nthr; ++t) {
    int s = 0;
    while (s < k && ang[s] < thr_host[t]) ++s;
    lces_host[t] = s;
  }
  return PPCA_OK;
}

// Certification support (reading R29): residual norms of Ritz pairs, one exact-fp32 SIMT
// pass (Y = X·Eᵀ, Z = YᵀX with fp64 split-K sums; no bf16 rounding of E or Y), all-reduced.
ppca_status ppca_ritz_residuals(ppca_ctx* h, const ppca_matrix* X, const float* E, int k, const double* theta_host,
                                double* res_host, double* res_gram_host) {
  if (!h) return PPCA_ERR_INVALID_ARG;
  Ctx* c = &h->c;
  enter(c);
  PPCA_TRY(check_matrix(c, X, k));
  if (!E || !theta_host || !res_host) return set_error(c, PPCA_ERR_INVALID_ARG, "null E / theta / res");
  const int64_t d = X->d;
  float* Y = (float*)scratch(c, S_Y, (size_t)std::max<int64_t>(1, X->n_local) * k * sizeof(float));
  float* Z = (float*)scratch(c, S_Z, (size_t)k * d * sizeof(float));
  double* buf = (double*)scratch(c, S_EVAL, (size_t)2 * k * sizeof(double));
  if (!Y || !Z || !buf) return set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
  if (X->n_local > 0) {
    PPCA_TRY(xw(c, X, 0, X->n_local, E, k, Y));
    PPCA_TRY(ytx(c, X, 0, X->n_local, Y, k, Z));
  } else {
    PPCA_TRY(check_cuda(c, cudaMemsetAsync(Z, 0, (size_t)k * d * sizeof(float), c->stream), "zero Z"));
  }
  PPCA_TRY(allreduce(c, Z, (size_t)k * d, false));
  PPCA_TRY(check_cuda(c, cudaMemcpyAsync(buf, theta_host, (size_t)k * sizeof(double), cudaMemcpyHostToDevice,
                                         c->stream), "copy theta"));
  PPCA_TRY(ritz_resid(c, Z, E, buf, k, d, buf + k));
  double* RG = nullptr;
  if (res_gram_host) {                                   // R R^T of the residual rows R_i = Z_i − θ_i E_i (in Z)
    RG = (double*)scratch(c, S_GRAM, (size_t)k * k * sizeof(double));
    if (!RG) return set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
    PPCA_TRY(resid_rows(c, Z, E, buf, k, d));
    PPCA_TRY(vec_gram(c, Z, k, d, RG));
  }
  PPCA_TRY(finish(c, "ppca_ritz_residuals"));
  if (cudaMemcpy(res_host, buf + k, (size_t)k * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess)
    return set_error(c, PPCA_ERR_CUDA, "copy residuals");
  if (res_gram_host && cudaMemcpy(res_gram_host, RG, (size_t)k * k * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess)
    return set_error(c, PPCA_ERR_CUDA, "copy residual Gram");
  return PPCA_OK;
}

ppca_status ppca_captured_variance(ppca_ctx* h, const ppca_matrix* X, const float* V, int m, double* var_host) {
  if (!h) return PPCA_ERR_INVALID_ARG;
  Ctx* c = &h->c;
  enter(c);
  PPCA_TRY(check_matrix(c, X, m));
  if (!V || !var_host) return set_error(c, PPCA_ERR_INVALID_ARG, "null V / output");
  double* S = (double*)scratch(c, S_S, (size_t)m * m * sizeof(double));
  PassPlan plan;
  PPCA_TRY(pass_prepare(c, X, m, &plan));
  PPCA_TRY(pass_gram(c, X, &plan, V, m, S));
  PPCA_TRY(allreduce(c, S, (size_t)m * m, true));
  PPCA_TRY(finish(c, "ppca_captured_variance"));
  std::vector<double> hs((size_t)m * m);
  if (cudaMemcpy(hs.data(), S, hs.size() * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess)
    return set_error(c, PPCA_ERR_CUDA, "copy S");
  for (int i = 0; i < m; ++i) var_host[i] = hs[(size_t)i * m + i];
  return PPCA_OK;
}

ppca_status ppca_gram(ppca_ctx* h, const ppca_matrix* X, double* G) {
  if (!h) return PPCA_ERR_INVALID_ARG;
  Ctx* c = &h->c;
  enter(c);
  PPCA_TRY(check_matrix(c, X, 1));
  if (!G) return set_error(c, PPCA_ERR_INVALID_ARG, "null G");
  const int64_t d = X->d;
  int ns = tn_pick_splits(c, d, d, X->n_local);
  double* P = (double*)scratch(c, S_PART, (size_t)ns * d * d * sizeof(double));
  if (!P) return set_error(c, PPCA_ERR_CUDA, "scratch alloc failed (d=%lld)", (long long)d);
  if (X->dtype == PPCA_F32)
    PPCA_TRY((launch_tn_splitk<float, float>(c, (const float*)X->data, X->ld, (const float*)X->data, X->ld, P, d, d,
                                             X->n_local, ns)));
  else if (X->dtype == PPCA_F32_SPLIT)
    PPCA_TRY((launch_tn_splitk<SplitF32, SplitF32>(c, (const SplitF32*)X->data, X->ld, (const SplitF32*)X->data,
                                                   X->ld, P, d, d, X->n_local, ns)));
  else
    PPCA_TRY((launch_tn_splitk<__nv_bfloat16, __nv_bfloat16>(c, (const __nv_bfloat16*)X->data, X->ld,
                                                             (const __nv_bfloat16*)X->data, X->ld, P, d, d,
                                                             X->n_local, ns)));
  PPCA_TRY(launch_reduce_splits_f64(c, P, ns, d * d, G));
  PPCA_TRY(allreduce(c, G, (size_t)d * d, true));
  return finish(c, "ppca_gram");
}

}  // extern "C"
