// pass_tc.cu — tcgen05 tensor-core streaming pass over X (impl 2; §8 rows a2 / a7).
//
// Two persistent, warp-specialised kernels (one CTA per SM):
//
//  xw_tc  (product 1, "refine mode" on its own):  Y_t = X_t·W'ᵀ for 128-row tiles X_t, accumulated in
//         TMEM over 64-column K chunks (UMMA M=128, N=m, K=16, bf16 operands, fp32 accumulate);
//         epilogue: S += Y_tᵀY_t (fp32 per tile, fp64 across tiles) and, in power mode, Yᵀ (bf16) out.
//  xty_tc (product 2):  Zᵀ[d-chunk] += X_tᵀ·Y_t, the same X bytes read as an MN-major A operand,
//         TMEM-resident partials per (d-group, row-group) work item, reduced in fixed order.
//
// Operands are bf16 in shared memory (SWIZZLE_128B atoms of 8 rows × 128 B).  An fp32 X is rounded
// to nearest bf16 on the way into shared memory by converter warps (LDG.128 → cvt.rn.bf16x2 → STS);
// a bf16 X is staged by TMA.  The tf32 kind would read fp32 X directly but the hardware truncates
// its inputs (profiles/r1_tc_microtest.txt), which biases Ritz values by ~-7e-4;
// bf16 RN is unbiased.  W' = RN_bf16(W) and the Rayleigh–Ritz step uses the Gram of W' (small.cu).
#include <cuda.h>
#include <cuda_bf16.h>
#include "pass.cuh"
#include "gemm_simt.cuh"
#include "tc_util.cuh"

namespace ppca {

using namespace tc;

// ============================================================================ host: tensor maps
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  }
  return fn;
}

// 2-D bf16 tensor map: inner dim (contiguous) `inner`, outer `outer`, row stride `ld` elements,
// box {64, box_rows}, SWIZZLE_128B, out-of-bounds elements read as zero.
static bool make_map_bf16(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint64_t ld,
                          uint32_t box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// byte offset of (row, byte) inside a stack of SW128 atoms (8 rows × 128 B, 1024 B each)
__device__ __forceinline__ uint32_t sw128(uint32_t row, uint32_t byte) {
  return (row >> 3) * 1024u + (row & 7u) * 128u + ((((byte >> 4) ^ (row & 7u)) << 4) | (byte & 15u));
}

__device__ __forceinline__ uint2 pack4_bf16(float4 v) {
  __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y);
  __nv_bfloat162 b = __floats2bfloat162_rn(v.z, v.w);
  return make_uint2(*reinterpret_cast<uint32_t*>(&a), *reinterpret_cast<uint32_t*>(&b));
}

// x − RN_bf16(x) for the four values packed in `hi`
__device__ __forceinline__ float4 residual_bf16(float4 v, uint2 hi) {
  return make_float4(v.x - __uint_as_float(hi.x << 16), v.y - __uint_as_float(hi.x & 0xffff0000u),
                     v.z - __uint_as_float(hi.y << 16), v.w - __uint_as_float(hi.y & 0xffff0000u));
}

// fp32 row segment [col, col+4) of row `r` (zero outside the matrix).  d % 8 == 0 on this path, so a
// segment is either wholly inside or wholly outside; nothing may touch the loaded value here, or the
// compiler has to wait for the load before issuing the next one.
__device__ __forceinline__ float4 ldg_x4(const float* __restrict__ X, int64_t ld, int64_t r, int64_t n, int64_t col,
                                         int64_t d) {
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  if (r < n && col < d) v = __ldcs(reinterpret_cast<const float4*>(X + r * ld + col));   // streamed once
  return v;
}

// ============================================================================ W' = W_hi + W_lo (bf16 pair)
// The vector set is split into two bf16 rows (hi = RN(W), lo = RN(W − hi)) stacked as [2·mp][d], so the
// span the tensor cores see is W to ~2^-17 (a single bf16 W would move a non-invariant span by ~2^-9
// and its Ritz values at first order).  Wr = hi + lo (fp32) is the operand's exact value, used for the
// Rayleigh–Ritz Gram and the lift.
__global__ void prep_w_kernel(const float* __restrict__ W, int m, int mp, int64_t d, __nv_bfloat16* __restrict__ Wb,
                              float* __restrict__ Wr) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)mp * d) return;
  int64_t i = e / d;
  float v = i < m ? W[e] : 0.f;
  __nv_bfloat16 hi = __float2bfloat16_rn(v);
  __nv_bfloat16 lo = __float2bfloat16_rn(v - __bfloat162float(hi));
  Wb[e] = hi;
  Wb[e + (int64_t)mp * d] = lo;
  if (i < m) Wr[e] = __bfloat162float(hi) + __bfloat162float(lo);
}

// S entry enumeration for the 128 epilogue threads: columns c1 = p and c2 = MP−1−p are paired
// (p = tid / TPP, TPP = 256/MP threads per pair); the pair's MP+1 upper-triangle entries
// (i ≤ c1 then i ≤ c2) are dealt round-robin over its TPP threads — balanced to ±1.
template <int MP>
__device__ __forceinline__ bool s_entry(int tid, int q, int& i, int& j) {
  constexpr int TPP = 256 / MP;
  const int p = tid / TPP, sub = tid % TPP;
  const int e = sub + q * TPP;
  if (p >= MP / 2 || e > MP) return false;
  if (e <= p) { i = e; j = p; } else { i = e - p - 1; j = MP - 1 - p; }
  return true;
}

// ============================================================================ wait profiling
// Per-role cycles spent in mbarrier waits (kernel A), read back by ppca_debug_wait_counters().
// Compiled in only with -DPPCA_WAIT_PROFILE (the counters cost registers in every role).
__device__ unsigned long long g_wait[16];
#ifdef PPCA_WAIT_PROFILE
#define TWAIT(bar, par, slot)                  \
  do {                                         \
    const long long _t0 = clock64();           \
    mbar_wait(bar, par);                       \
    wacc[slot] += clock64() - _t0;             \
  } while (0)
#else
#define TWAIT(bar, par, slot) mbar_wait(bar, par)
#endif

// ============================================================================ kernel A: Y = X·W'ᵀ, S = YᵀY
namespace ka {
constexpr int BM = 128;          // rows per tile (UMMA M)
constexpr int BK = 64;           // bf16 K elements per chunk (one 128-B swizzle row)
constexpr int NST = 4;           // smem pipeline stages
constexpr int NCONV = 8;         // converter warps (fp32 X)
constexpr int W_EPI0 = 0;        // warps 0..3: epilogue (TMEM lane quadrants 0..3)
constexpr int W_CONV0 = 4;       // warps 4..11: converters
constexpr int W_PROD = 12;       // control warp: lane 0 W' TMA, lane 1 X TMA (bf16 X), lane 2 MMA issue
constexpr int W_MMA = 12;        // TMEM owner (same warp)
constexpr int NTHREADS = 13 * 32;
constexpr uint32_t XST = BM * 128;   // X stage bytes
// ring depths: X stages (bf16 pair for fp32 X) and W' stages ([W_hi; W_lo], 2·MP rows × 128 B)
__host__ __device__ constexpr int nst(int MP, bool xbf16) { return xbf16 ? 4 : (MP <= 64 ? 3 : 2); }
__host__ __device__ constexpr int nws(int MP) { return MP <= 64 ? 4 : 2; }
__host__ __device__ constexpr size_t smem_bytes(int MP, bool xbf16) {
  return 1024 + (size_t)nst(MP, xbf16) * (xbf16 ? XST : 2 * XST) + (size_t)nws(MP) * 2 * MP * 128 +
         (size_t)BM * (MP + 4) * 4 + 16 + 512;
}
}  // namespace ka
#define KA_NWS(MP, XBF16) ka::nws(MP)

struct KAParams {
  const void* X;          // fp32 or bf16 [n][ld]
  int64_t n, d, ld;
  int m, mp;              // m, m padded to a multiple of 16
  int64_t ntiles, nk;     // row tiles, K chunks
  __nv_bfloat16* YT;      // optional Yᵀ out, bf16 [mp][ldyt]
  int64_t ldyt;
  double* Spart;          // [gridDim.x][mp][mp] fp64 per-CTA partials
};

template <int MP, bool XBF16>
__global__ void __launch_bounds__(ka::NTHREADS, 1)
    xw_tc_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX, KAParams p) {
  using namespace ka;
  // fp32 X is staged as a bf16 pair too (X_hi at +0, X_lo at +XST): Y = X_hi·W_hiᵀ + X_lo·W_hiᵀ + X_hi·W_loᵀ
  constexpr uint32_t XSTG = XBF16 ? XST : 2 * XST;
  constexpr int NST = ka::nst(MP, XBF16);          // X smem pipeline stages
  static_assert(ka::smem_bytes(MP, XBF16) <= 227 * 1024, "kernel A shared memory budget");
  constexpr int NB = 2 * MP;                       // UMMA N: [W_hi; W_lo]
  constexpr uint32_t WST = NB * 128;
  constexpr int NTB = NB <= 128 ? 4 : 2;           // TMEM accumulator ring depth (MMA runs ahead of the epilogue)
  constexpr uint32_t TCOLS = (NTB * NB <= 32) ? 32 : (NTB * NB <= 64 ? 64 : (NTB * NB <= 128 ? 128 : (NTB * NB <= 256 ? 256 : 512)));
  constexpr bool SREG = MP <= 64;                  // keep S partials in registers
  constexpr int YS_LD = MP + 4;                    // 16-B aligned rows for LDS.128
  // W' chunks have their own, deeper ring: they come from L2 with TMA latency and must not wait for the
  // X stage of the same chunk to drain (the X ring would otherwise serialise on the W round trip).
  constexpr int NWS = KA_NWS(MP, XBF16);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sX = sm;                                  // NST × XSTG
  uint8_t* sW = sX + NST * XSTG;                     // NWS × WST
  float* Ys = reinterpret_cast<float*>(sW + NWS * WST);   // BM × YS_LD
  uint64_t* bars = reinterpret_cast<uint64_t*>(Ys + BM * YS_LD + 2);
  uint64_t* full = bars;
  uint64_t* empty = bars + NST;
  uint64_t* tfull = bars + 2 * NST;
  uint64_t* tempty = bars + 2 * NST + NTB;
  uint64_t* wfull = bars + 2 * NST + 2 * NTB;
  uint64_t* wempty = wfull + NWS;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(wempty + NWS);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef PPCA_WAIT_PROFILE
  long long wacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const long long kstart = clock64();
#endif
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], XBF16 ? 1 : NCONV);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < NWS; ++s) {
      mbar_init(&wfull[s], 1);
      mbar_init(&wempty[s], 1);
    }
    for (int b = 0; b < NTB; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
    }
    fence_barrier_init();
  }
  if (warp == W_PROD && lane == 0) {
    tma_prefetch_desc(&tmW);
    if (XBF16) tma_prefetch_desc(&tmX);
  }
  if (warp == W_MMA) tmem_alloc<TCOLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int64_t t0 = blockIdx.x, tstep = gridDim.x;

  if (warp == W_PROD) {
    // ------------------------------------------------------------------ TMA producers
    if (lane == 0) {                                 // W' ring
      uint32_t it = 0;
      for (int64_t t = t0; t < p.ntiles; t += tstep)
        for (int64_t kc = 0; kc < p.nk; ++kc, ++it) {
          const uint32_t s = it % NWS, ph = (it / NWS) & 1;
          TWAIT(&wempty[s], ph ^ 1, 0);
          mbar_arrive_expect_tx(&wfull[s], WST);
          tma_load_2d(sW + s * WST, &tmW, &wfull[s], (int32_t)(kc * BK), 0);
        }
    } else if (XBF16 && lane == 1) {                 // X ring (bf16 X)
      uint64_t pol = policy_evict_first();
      uint32_t it = 0;
      for (int64_t t = t0; t < p.ntiles; t += tstep)
        for (int64_t kc = 0; kc < p.nk; ++kc, ++it) {
          const uint32_t s = it % NST, ph = (it / NST) & 1;
          TWAIT(&empty[s], ph ^ 1, 1);
          mbar_arrive_expect_tx(&full[s], XST);
          tma_load_2d_hint(sX + s * XSTG, &tmX, &full[s], (int32_t)(kc * BK), (int32_t)(t * BM), pol);
        }
    } else if (lane == 2) {
    // ------------------------------------------------------------------ MMA issuer (one thread)
    constexpr uint32_t ID = idesc(FMT_BF16, FMT_BF16, BM, NB, 0, 0);
    uint32_t it = 0, tt = 0;
    for (int64_t t = t0; t < p.ntiles; t += tstep, ++tt) {
      const uint32_t b = tt % NTB, tph = (tt / NTB) & 1;
      TWAIT(&tempty[b], tph ^ 1, 2);
      tc_fence_after();
      const uint32_t dcol = tmem + b * NB;
      for (int64_t kc = 0; kc < p.nk; ++kc, ++it) {
        const uint32_t s = it % NST, ph = (it / NST) & 1;
        const uint32_t ws = it % NWS, wph = (it / NWS) & 1;
        TWAIT(&wfull[ws], wph, 3);
        TWAIT(&full[s], ph, 4);
        tc_fence_after();
        {
          const uint32_t xa = smem_u32(sX + s * XSTG), wa = smem_u32(sW + ws * WST);
          constexpr uint32_t ID_HI = idesc(FMT_BF16, FMT_BF16, BM, MP, 0, 0);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            // [hi | lo] columns += X_hi·[W_hi; W_lo]ᵀ
            mma_bf16(dcol, smem_desc_sw128(xa + kk * 32, 16, 1024), smem_desc_sw128(wa + kk * 32, 16, 1024), ID,
                     (kc | kk) != 0);
            // hi columns += X_lo·W_hiᵀ  (fp32 X only)
            if (!XBF16)
              mma_bf16(dcol, smem_desc_sw128(xa + XST + kk * 32, 16, 1024), smem_desc_sw128(wa + kk * 32, 16, 1024),
                       ID_HI, 1);
          }
          mma_commit(&empty[s]);
          mma_commit(&wempty[ws]);
        }
      }
      mma_commit(&tfull[b]);
    }
    }
  } else if (warp >= W_CONV0 && warp < W_CONV0 + NCONV) {
    // ------------------------------------------------------------------ fp32 → bf16 converters
    if (!XBF16) {
      const float* X = reinterpret_cast<const float*>(p.X);
      const int cw = warp - W_CONV0;
      const int sub = lane >> 4, cl = lane & 15;
      // chunk ci of this CTA = (tile t0 + (ci / nk)·tstep, K chunk ci % nk) — the producer/MMA order.
      // Three register buffers rotate so two chunks of loads are in flight while one is stored.
      const int64_t nchunks = ((p.ntiles - t0 + tstep - 1) / tstep) * p.nk;
      // load cursor (tile, kc) and store cursor (stage, phase) advance incrementally (no 64-bit divides)
      int64_t lt = t0, lk = 0;
      uint32_t ss = 0, sph = 0;
      auto load = [&](int64_t ci, float4 (&r)[8]) {
        if (ci >= nchunks) return;
        const int64_t row0 = lt * BM + cw * 16 + sub;
        const int64_t col = lk * BK + cl * 4;
        const float* base = X + row0 * p.ld + col;
        const bool colok = col < p.d;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
          if (colok && row0 + 2 * i < p.n) v = __ldcs(reinterpret_cast<const float4*>(base + 2 * i * p.ld));
          r[i] = v;
        }
        if (++lk == p.nk) { lk = 0; lt += tstep; }
      };
      auto store = [&](int64_t ci, const float4 (&r)[8]) {
        (void)ci;
        const uint32_t s = ss, ph = sph;
        if (++ss == NST) { ss = 0; sph ^= 1; }
        TWAIT(&empty[s], ph ^ 1, 5);
        uint8_t* st = sX + s * XSTG;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint32_t rr = cw * 16 + 2 * i + sub;
          const uint32_t off = sw128(rr, cl * 8);
          uint2 hi = pack4_bf16(r[i]);
          *reinterpret_cast<uint2*>(st + off) = hi;
          *reinterpret_cast<uint2*>(st + XST + off) = pack4_bf16(residual_bf16(r[i], hi));
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[s]);
      };
      float4 A[8], B[8], Cb[8];
      load(0, A);
      load(1, B);
      for (int64_t ci = 0; ci < nchunks; ci += 3) {
        load(ci + 2, Cb);
        store(ci, A);
        if (ci + 1 >= nchunks) break;
        load(ci + 3, A);
        store(ci + 1, B);
        if (ci + 2 >= nchunks) break;
        load(ci + 4, B);
        store(ci + 2, Cb);
      }
    }
  } else if (warp < 4) {
    // ------------------------------------------------------------------ epilogue (128 threads)
    // S = Σ_tiles Y_tᵀY_t: thread t owns 4×4 blocks (bi ≤ bj) b = t, t+128, … of the upper triangle;
    // per tile each block is 128 rows × (2 LDS.128 + 16 FMA) in fp32, then added to fp64 accumulators.
    const int tid = threadIdx.x;                     // 0..127 = TMEM lane = tile row
    constexpr int NBK = MP / 4, NBLK = NBK * (NBK + 1) / 2, MAXB = (NBLK + 127) / 128;
    int bi_[MAXB], bj_[MAXB];
#pragma unroll
    for (int q = 0; q < MAXB; ++q) {
      int b = tid + 128 * q, bi = 0;
      bi_[q] = -1;
      bj_[q] = 0;
      if (b < NBLK) {
        while (b >= NBK - bi) { b -= NBK - bi; ++bi; }
        bi_[q] = bi;
        bj_[q] = bi + b;
      }
    }
    double acc[SREG ? MAXB : 1][16];
#pragma unroll
    for (int q = 0; q < (SREG ? MAXB : 1); ++q)
#pragma unroll
      for (int e = 0; e < 16; ++e) acc[q][e] = 0.0;
    double* Sp = p.Spart + (int64_t)blockIdx.x * MP * MP;
    if (!SREG)
      for (int q = 0; q < MAXB; ++q)
        if (bi_[q] >= 0)
          for (int e = 0; e < 16; ++e) Sp[(4 * bi_[q] + e / 4) * MP + 4 * bj_[q] + e % 4] = 0.0;
    uint32_t tt = 0;
    for (int64_t t = t0; t < p.ntiles; t += tstep, ++tt) {
      const uint32_t b = tt % NTB, tph = (tt / NTB) & 1;
      TWAIT(&tfull[b], tph, 6);
      tc_fence_after();
      const int64_t grow = t * BM + tid;
#pragma unroll 1
      for (int c0 = 0; c0 < MP; c0 += 16) {
        float v[16], w[16];
        const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + b * NB + c0;
        tmem_ld16(ta, v);          // X'·W_hiᵀ
        tmem_ld16(ta + MP, w);     // X'·W_loᵀ
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] += w[j];
#pragma unroll
        for (int j = 0; j < 16; j += 4)
          *reinterpret_cast<float4*>(Ys + tid * YS_LD + c0 + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        if (p.YT && grow < p.ldyt) {       // Yᵀ as a bf16 pair [Y_hi; Y_lo] (rows ≥ n are zero)
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const __nv_bfloat16 hi = __float2bfloat16_rn(v[j]);
            p.YT[(int64_t)(c0 + j) * p.ldyt + grow] = hi;
            p.YT[(int64_t)(MP + c0 + j) * p.ldyt + grow] = __float2bfloat16_rn(v[j] - __bfloat162float(hi));
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[b]);
      asm volatile("bar.sync 1, 128;" ::: "memory");
#pragma unroll
      for (int q = 0; q < MAXB; ++q) {
        if (bi_[q] < 0) continue;
        float s[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) s[e] = 0.f;
        const float* ya = Ys + 4 * bi_[q];
        const float* yb = Ys + 4 * bj_[q];
#pragma unroll 4
        for (int r = 0; r < BM; ++r) {
          const float4 a = *reinterpret_cast<const float4*>(ya + r * YS_LD);
          const float4 c = *reinterpret_cast<const float4*>(yb + r * YS_LD);
          const float av[4] = {a.x, a.y, a.z, a.w}, cv[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
          for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y) s[x * 4 + y] = fmaf(av[x], cv[y], s[x * 4 + y]);
        }
        if (SREG) {
#pragma unroll
          for (int e = 0; e < 16; ++e) acc[SREG ? q : 0][e] += (double)s[e];
        } else {
#pragma unroll
          for (int e = 0; e < 16; ++e) Sp[(4 * bi_[q] + e / 4) * MP + 4 * bj_[q] + e % 4] += (double)s[e];
        }
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
    }
    if (SREG)
#pragma unroll
      for (int q = 0; q < MAXB; ++q)
        if (bi_[q] >= 0)
#pragma unroll
          for (int e = 0; e < 16; ++e)
            Sp[(4 * bi_[q] + e / 4) * MP + 4 * bj_[q] + e % 4] = acc[SREG ? q : 0][e];
  }
  tc_fence_before();
  __syncthreads();
#ifdef PPCA_WAIT_PROFILE
  if (lane == 0) {
    for (int k = 0; k < 7; ++k)
      if (wacc[k]) atomicAdd(&g_wait[k], (unsigned long long)wacc[k]);
    if (threadIdx.x == 0) atomicAdd(&g_wait[15], (unsigned long long)(clock64() - kstart));
  }
#endif
  if (warp == W_MMA) tmem_dealloc<TCOLS>(tmem);
}

// S[i][j] = S[j][i] = Σ_cta Spart[cta][pair(i,j)]  (fixed order, fp64)
// Block = 32 outputs (lanes) × 8 warps; warp w sums partials c ≡ w (mod 8), then the 8 warp sums are
// added in warp order — a fixed order, so the result is deterministic.
__global__ void __launch_bounds__(256) reduce_spart_kernel(const double* __restrict__ Spart, int nparts, int mp, int m,
                                                           double* __restrict__ S) {
  __shared__ double part[8][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int e = blockIdx.x * 32 + lane;
  double s = 0.0;
  if (e < m * m) {
    const int i = e / m, j = e % m;
    const int idx = min(i, j) * mp + max(i, j);   // partials hold the upper triangle, dense [mp][mp]
    for (int c = warp; c < nparts; c += 8) s += Spart[(int64_t)c * mp * mp + idx];
  }
  part[warp][lane] = s;
  __syncthreads();
  if (warp == 0 && e < m * m) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += part[w][lane];
    S[e] = t;
  }
}

// ============================================================================ kernel B (tc_xty.cuh)
#include "tc_xty.cuh"

// Z[j][x] = Σ_g Zp[g][x][j]   (fixed order over row groups)
// Block (x, 32 consecutive j): lanes read 128 contiguous bytes of a partial row; warp w sums row groups
// g ≡ w (mod 8); the 8 warp sums are added in warp order (deterministic).
__global__ void __launch_bounds__(256) reduce_zp_kernel(const float* __restrict__ Zp, int64_t nrg, int64_t dpad, int mp,
                                                        int m, int64_t d, float* __restrict__ Z) {
  __shared__ double part[8][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t x = blockIdx.x;
  const int j = blockIdx.y * 32 + lane;
  double s = 0.0;
  if (j < m)
    for (int64_t g = warp; g < nrg; g += 8) s += Zp[(g * dpad + x) * mp + j];
  part[warp][lane] = s;
  __syncthreads();
  if (warp == 0 && j < m) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += part[w][lane];
    Z[(int64_t)j * d + x] = (float)t;
  }
}

// ============================================================================ host side
struct TcState {
  int sm = 148;
};

static int pad16(int m) { return (m + 15) & ~15; }

template <int MP, bool XBF16>
static ppca_status launch_ka(Ctx* c, const CUtensorMap& tmW, const CUtensorMap& tmX, const KAParams& kp, int grid) {
  const size_t smem = ka::smem_bytes(MP, XBF16);
  auto kern = xw_tc_kernel<MP, XBF16>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<<<grid, ka::NTHREADS, smem, c->stream>>>(tmW, tmX, kp);
  PPCA_LAUNCH_CHECK(c, "xw_tc_kernel");
  return PPCA_OK;
}

template <int MP, bool XBF16>
static ppca_status launch_kb(Ctx* c, const CUtensorMap& tmYT, const CUtensorMap& tmX, const KBParams& bp, int grid) {
  const size_t smem = kb::Cfg<MP>::SMEM;
  auto kern = xty_tc_kernel<MP, XBF16>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<<<grid, kb::NTHREADS, smem, c->stream>>>(tmYT, tmX, bp);
  PPCA_LAUNCH_CHECK(c, "xty_tc_kernel");
  return PPCA_OK;
}

template <bool XBF16>
static ppca_status dispatch_ka(Ctx* c, int mp, const CUtensorMap& tmW, const CUtensorMap& tmX, const KAParams& kp,
                               int grid) {
  switch (mp) {
    case 16: return launch_ka<16, XBF16>(c, tmW, tmX, kp, grid);
    case 32: return launch_ka<32, XBF16>(c, tmW, tmX, kp, grid);
    case 48: return launch_ka<48, XBF16>(c, tmW, tmX, kp, grid);
    case 64: return launch_ka<64, XBF16>(c, tmW, tmX, kp, grid);
    case 80: return launch_ka<80, XBF16>(c, tmW, tmX, kp, grid);
    case 96: return launch_ka<96, XBF16>(c, tmW, tmX, kp, grid);
    case 112: return launch_ka<112, XBF16>(c, tmW, tmX, kp, grid);
    case 128: return launch_ka<128, XBF16>(c, tmW, tmX, kp, grid);
  }
  return set_error(c, PPCA_ERR_UNSUPPORTED, "tcgen05 pass: m=%d unsupported", mp);
}

template <bool XBF16>
static ppca_status dispatch_kb(Ctx* c, int mp, const CUtensorMap& tmYT, const CUtensorMap& tmX, const KBParams& bp,
                               int grid) {
  switch (mp) {
    case 16: return launch_kb<16, XBF16>(c, tmYT, tmX, bp, grid);
    case 32: return launch_kb<32, XBF16>(c, tmYT, tmX, bp, grid);
    case 48: return launch_kb<48, XBF16>(c, tmYT, tmX, bp, grid);
    case 64: return launch_kb<64, XBF16>(c, tmYT, tmX, bp, grid);
    case 80: return launch_kb<80, XBF16>(c, tmYT, tmX, bp, grid);
    case 96: return launch_kb<96, XBF16>(c, tmYT, tmX, bp, grid);
    case 112: return launch_kb<112, XBF16>(c, tmYT, tmX, bp, grid);
    case 128: return launch_kb<128, XBF16>(c, tmYT, tmX, bp, grid);
  }
  return set_error(c, PPCA_ERR_UNSUPPORTED, "tcgen05 pass: m=%d unsupported", mp);
}

ppca_status pass_tc_prepare(Ctx* c, const ppca_matrix* X, int m, PassPlan* plan) {
  if (!encode_fn()) return set_error(c, PPCA_ERR_UNSUPPORTED, "cuTensorMapEncodeTiled unavailable");
  if (X->d % 8 != 0 || X->d < 64) return set_error(c, PPCA_ERR_UNSUPPORTED, "tcgen05 pass needs d %% 8 == 0, d >= 64");
  if (m > 128 || m < 1) return set_error(c, PPCA_ERR_UNSUPPORTED, "tcgen05 pass needs m <= 128");
  if (X->n_local < 128) return set_error(c, PPCA_ERR_UNSUPPORTED, "tcgen05 pass needs >= 128 local rows");
  if (X->dtype == PPCA_BF16 && (reinterpret_cast<uintptr_t>(X->data) % 16)) return set_error(c, PPCA_ERR_UNSUPPORTED, "X not 16B aligned");
  if (X->dtype == PPCA_F32 && (reinterpret_cast<uintptr_t>(X->data) % 16)) return set_error(c, PPCA_ERR_UNSUPPORTED, "X not 16B aligned");
  plan->impl = 2;
  return PPCA_OK;
}

// W' (bf16 + its fp32 value copy) → S_TC1;  returns pointers
static ppca_status prep_w(Ctx* c, const float* W, int m, int mp, int64_t d, __nv_bfloat16** Wb, float** Wr) {
  uint8_t* buf = (uint8_t*)scratch(c, S_TC1, (size_t)2 * mp * d * 2 + (size_t)m * d * 4 + 256);
  if (!buf) return set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
  *Wb = reinterpret_cast<__nv_bfloat16*>(buf);
  *Wr = reinterpret_cast<float*>(buf + (((size_t)2 * mp * d * 2 + 255) & ~(size_t)255));
  prep_w_kernel<<<(unsigned)ceil_div((int64_t)mp * d, 256), 256, 0, c->stream>>>(W, m, mp, d, *Wb, *Wr);
  PPCA_LAUNCH_CHECK(c, "prep_w");
  return PPCA_OK;
}

static ppca_status run_ka(Ctx* c, const ppca_matrix* X, const __nv_bfloat16* Wb, int m, int mp, double* S,
                          __nv_bfloat16* YT, int64_t ldyt) {
  CUtensorMap tmW, tmX;
  if (!make_map_bf16(&tmW, Wb, X->d, 2 * mp, X->d, 2 * mp)) return set_error(c, PPCA_ERR_CUDA, "tensor map W failed");
  if (X->dtype == PPCA_BF16) {
    if (!make_map_bf16(&tmX, X->data, X->d, X->n_local, X->ld, 128)) return set_error(c, PPCA_ERR_CUDA, "tensor map X failed");
  } else {
    tmX = tmW;   // unused
  }
  KAParams kp;
  kp.X = X->data; kp.n = X->n_local; kp.d = X->d; kp.ld = X->ld; kp.m = m; kp.mp = mp;
  kp.ntiles = ceil_div(X->n_local, ka::BM);
  kp.nk = ceil_div(X->d, ka::BK);
  kp.YT = YT; kp.ldyt = ldyt;
  int grid = (int)std::min<int64_t>(c->sm_count, kp.ntiles);
  double* Spart = (double*)scratch(c, S_TC0, (size_t)grid * mp * mp * sizeof(double));
  if (!Spart) return set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
  kp.Spart = Spart;
  PPCA_TRY(X->dtype == PPCA_BF16 ? dispatch_ka<true>(c, mp, tmW, tmX, kp, grid) : dispatch_ka<false>(c, mp, tmW, tmX, kp, grid));
  reduce_spart_kernel<<<(unsigned)ceil_div(m * m, 32), 256, 0, c->stream>>>(Spart, grid, mp, m, S);
  PPCA_LAUNCH_CHECK(c, "reduce_spart");
  return PPCA_OK;
}

ppca_status pass_tc_gram(Ctx* c, const ppca_matrix* X, const PassPlan* plan, const float* W, int m, double* S) {
  const int mp = pad16(m);
  __nv_bfloat16* Wb;
  float* Wr;
  PPCA_TRY(prep_w(c, W, m, mp, X->d, &Wb, &Wr));
  const_cast<PassPlan*>(plan)->Wop = Wr;
  return run_ka(c, X, Wb, m, mp, S, nullptr, 0);
}

ppca_status pass_tc_power(Ctx* c, const ppca_matrix* X, const PassPlan* plan, const float* W, int m, float* Z, double* S) {
  const int mp = pad16(m);
  const int64_t n = X->n_local, d = X->d;
  __nv_bfloat16* Wb;
  float* Wr;
  PPCA_TRY(prep_w(c, W, m, mp, d, &Wb, &Wr));
  const_cast<PassPlan*>(plan)->Wop = Wr;
  // Yᵀ as a bf16 pair [Y_hi; Y_lo], [2·mp][ldyt]; kernel A writes every row and column < ldyt
  const int64_t ldyt = ceil_div(n, 64) * 64;
  __nv_bfloat16* YT = (__nv_bfloat16*)scratch(c, S_Y, (size_t)2 * mp * ldyt * 2);
  if (!YT) return set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
  PPCA_TRY(run_ka(c, X, Wb, m, mp, S, YT, ldyt));
  // kernel B
  const int nc = mp <= 64 ? 2 : 1;
  KBParams bp;
  bp.X = X->data; bp.n = n; bp.d = d; bp.ld = X->ld; bp.m = m; bp.mp = mp;
  bp.ndg = ceil_div(d, nc * 128);
  int64_t want = std::max<int64_t>(1, ceil_div(4 * (int64_t)c->sm_count, bp.ndg));
  int64_t rpg = ceil_div(ceil_div(n, want), kb::KR) * kb::KR;
  rpg = std::max<int64_t>(rpg, kb::KR);
  bp.rows_per_rg = rpg;
  bp.nrg = ceil_div(n, rpg);
  const int64_t dpad = bp.ndg * nc * 128;
  float* Zp = (float*)scratch(c, S_PART, (size_t)bp.nrg * dpad * mp * sizeof(float));
  if (!Zp) return set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
  bp.Zp = Zp;
  CUtensorMap tmYT, tmX;
  if (!make_map_bf16(&tmYT, YT, ldyt, 2 * mp, ldyt, 2 * mp)) return set_error(c, PPCA_ERR_CUDA, "tensor map YT failed");
  if (X->dtype == PPCA_BF16) {
    if (!make_map_bf16(&tmX, X->data, d, n, X->ld, kb::KR)) return set_error(c, PPCA_ERR_CUDA, "tensor map X failed");
  } else {
    tmX = tmYT;
  }
  const int grid = (int)std::min<int64_t>(c->sm_count, bp.ndg * bp.nrg);
  PPCA_TRY(X->dtype == PPCA_BF16 ? dispatch_kb<true>(c, mp, tmYT, tmX, bp, grid) : dispatch_kb<false>(c, mp, tmYT, tmX, bp, grid));
  reduce_zp_kernel<<<dim3((unsigned)d, (unsigned)ceil_div(m, 32)), 256, 0, c->stream>>>(Zp, bp.nrg, dpad, mp, m, d, Z);
  PPCA_LAUNCH_CHECK(c, "reduce_zp");
  return PPCA_OK;
}

void pass_tc_release(Ctx*) {}

ppca_status debug_wait_counters(unsigned long long* out16) {
  cudaDeviceSynchronize();
  if (cudaMemcpyFromSymbol(out16, g_wait, 16 * sizeof(unsigned long long)) != cudaSuccess) return PPCA_ERR_CUDA;
  unsigned long long z[16] = {};
  cudaMemcpyToSymbol(g_wait, z, sizeof z);
  return PPCA_OK;
}

}  // namespace ppca
