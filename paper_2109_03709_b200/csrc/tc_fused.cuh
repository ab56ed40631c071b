// tc_fused.cuh — single-read power pass (§8 row a2): Y = X·W'ᵀ, S = YᵀY and Zᵀ = X_hiᵀ·[Y_hi; Y_lo] in ONE
// persistent kernel, so the hi plane of X is re-read from L2 right after it streamed from HBM instead of a
// second HBM pass (kernel B).
//
// Why cross-SM: Zᵀ for d = 1024, m = 64 is 256 KB fp32 — all of one SM's TMEM — so one SM cannot hold it
// next to the Y accumulators.  The CTAs are grouped: CTA (r, g), g < ndg d-groups of DG = 256 columns,
// r < nrg row groups.  The tiles of row group r are dealt round-robin to its ndg CTAs for product 1
// ("A-work": HBM stream of both planes, Y, S, Yᵀ to global, then a per-tile ready flag); every CTA of the
// group then accumulates product 2 for its own d-group over ALL the group's tiles ("B-work": waits for the
// tile's flag, TMA-loads Yᵀ and X_hi[tile, d-group] — which a sibling has just pulled through L2).
// Rounds keep the siblings in step: round ρ = the ndg tiles ρ·ndg + j; A-work of round ρ precedes B-work of
// round ρ in every CTA.  All CTAs are co-resident (cooperative launch, ≤ one per SM), so the flag waits
// terminate; each wait is also bounded (kFlagTimeoutNs → DEV_TIMEOUT).
//
// TMEM (512 columns): Y accumulator [0, 128) (one buffer), S [128, 256), Zᵀ [256, 512) (two 128-row d-chunks
// × N = 128 = [Y_hi; Y_lo]).  Shared memory (default configuration): A ring 2 × 32 KB (hi + lo planes), W' ring
// 2 × 16 KB, B ring 2 × 48 KB (X_hi 64 rows × 256 columns + Y 64 rows × [Y_hi | Y_lo], both MN-major).  S = YᵀY of an own tile
// is chained on the B-stream from the same staged Y rows (no separate Y operand tile).
// The Y rows go through global memory row-major (one 256-byte store per row) for the siblings.
// Numerics are those of kernels A2 + B: the same MMAs in the same order per tile.
#pragma once

namespace kf {
constexpr int BM = 128, BK = 64, KSEG = 16, SFLUSH = 8;
constexpr int MP = 64, NB = 2 * MP;            // m padded; product-1 N and product-2 N ([Y_hi; Y_lo])
constexpr int DG = 256, NC = DG / 128;         // d-group width, 128-row d chunks per group
constexpr int KR = 64;                         // rows per B stage (64: 12 % faster than 32 on C3, measured)
constexpr uint32_t XPL = BM * 128;             // one bf16 plane chunk: 128 rows × 64 columns
constexpr uint32_t WST = NB * 128;             // W' chunk: 128 rows ([W_hi; W_lo]) × 64 columns
constexpr uint32_t BBLK = KR * 128;            // KR rows × 64 columns (SW128 atoms of 8 rows)
constexpr uint32_t BX = NC * 2 * BBLK;         // X_hi part of a B stage (256 columns)
constexpr uint32_t BY = 2 * BBLK;              // Y part of a B stage: KR rows × [Y_hi | Y_lo] (MN-major)
constexpr int W_WPROD = 4, W_XPROD = 5, W_BPROD = 6, W_MMA = 7;
constexpr int NTHREADS = 8 * 32;
constexpr uint32_t TY = 0, TS = 128, TZ = 256;   // TMEM column bases
}  // namespace kf

struct KFParams {
  int64_t n, d;
  int m;
  int64_t ntiles, nk, nseg;
  int ndg, nrg;
  int64_t tiles_per_rg;          // row group r: tiles [r·tpr, min(ntiles, (r+1)·tpr))
  __nv_bfloat16* Yrm;            // Y as row-major bf16 pairs [n_pad][Y_hi(64) | Y_lo(64)] (MN-major B operand)
  int64_t nrow_pad;
  double* Spart;                 // [grid][2·MP][MP]
  float* Zp;                     // [nrg][ndg·DG][MP]
  int* flags;                    // [ntiles] = epoch when the tile's Yᵀ rows are written
  int epoch;
  int pf;                        // A-stream L2 prefetch distance in chunks (0 = off)
  int dbg;                       // experiment switches (PPCA_DBG; 0 in production): 1 skip B-stream
  int hi_policy;                 // L2 policy of the A-stream's hi plane: 0 evict_last, 1 normal, 2 evict_first
  int lag;                       // > 0: the A-stream starts round ρ only once the B-stream finished round ρ−lag−1
                                 // (bounds the X_hi rounds waiting in L2 for their re-read); 0: unbounded
  int* err;                      // device error word: DEV_TIMEOUT if a sibling's tile flag never arrives
};

// Bound on one inter-CTA wait (a sibling's tile flag).  The kernel is launched cooperatively (all CTAs
// co-resident, or the launch fails and the two-kernel pass runs instead), so the wait normally lasts well
// under a pass; the bound turns a broken residency assumption into PPCA_ERR_CUDA instead of a hang.
constexpr uint64_t kFlagTimeoutNs = 2000000000ull;

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

template <int XM, int NSTA, int NWS, int NSTB>
__global__ void __launch_bounds__(kf::NTHREADS, 1)
    xwz_fused_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                     const __grid_constant__ CUtensorMap tmXlo, const __grid_constant__ CUtensorMap tmXb,
                     const __grid_constant__ CUtensorMap tmY, KFParams p) {
  using namespace kf;
  constexpr bool LO = XM == 2;
  constexpr uint32_t XSTG = LO ? 2 * XPL : XPL;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = sm;                               // NSTA × XSTG
  uint8_t* sW = sA + NSTA * XSTG;                 // NWS × WST
  uint8_t* sB = sW + NWS * WST;                   // NSTB × (BX + BY)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + NSTB * (BX + BY));
  uint64_t* afull = bars;                         // NSTA
  uint64_t* aempty = afull + NSTA;
  uint64_t* wfull = aempty + NSTA;                // NWS
  uint64_t* wempty = wfull + NWS;
  uint64_t* bfull = wempty + NWS;                 // NSTB
  uint64_t* bempty = bfull + NSTB;
  uint64_t* tfull = bempty + NSTB;                // Y accumulator ready / drained
  uint64_t* tempty = tfull + 1;
  uint64_t* sempty = tempty + 1;                  // S accumulator drained (4 epilogue warps)
  uint64_t* sfull = sempty + 1;                   // S chain of an own tile complete
  uint64_t* zfull = sfull + 1;                    // all product-2 MMAs complete
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(zfull + 1);
  volatile int* bdone = reinterpret_cast<volatile int*>(tmem_slot + 1);   // rounds the B-stream has loaded

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = blockIdx.x % p.ndg, r = blockIdx.x / p.ndg;
  const int64_t tb = (int64_t)r * p.tiles_per_rg, te = min(p.ntiles, tb + p.tiles_per_rg);
  const int64_t nrounds = te > tb ? (te - tb + p.ndg - 1) / p.ndg : 0;
  // own (A-work) tile of round ρ, or -1
  auto own_tile = [&](int64_t rho) -> int64_t {
    const int64_t t = tb + rho * p.ndg + g;
    return t < te ? t : -1;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTA; ++s) { mbar_init(&afull[s], 1); mbar_init(&aempty[s], 1); }
    for (int s = 0; s < NWS; ++s) { mbar_init(&wfull[s], 1); mbar_init(&wempty[s], 1); }
    for (int s = 0; s < NSTB; ++s) { mbar_init(&bfull[s], 1); mbar_init(&bempty[s], 1); }
    mbar_init(tfull, 1);
    mbar_init(tempty, 4);
    mbar_init(sempty, 4);
    mbar_init(sfull, 1);
    mbar_init(zfull, 1);
    *bdone = 0;
    fence_barrier_init();
  }
  if (warp == W_XPROD && lane == 0) {
    tma_prefetch_desc(&tmW);
    tma_prefetch_desc(&tmX);
    if (LO) tma_prefetch_desc(&tmXlo);
    tma_prefetch_desc(&tmXb);
    tma_prefetch_desc(&tmY);
  }
  if (warp == W_MMA) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == W_WPROD) {
    if (lane == 0) {
      uint32_t it = 0;
      for (int64_t rho = 0; rho < nrounds; ++rho) {
        if (own_tile(rho) < 0) continue;
        for (int64_t kc = 0; kc < p.nk; ++kc, ++it) {
          const uint32_t s = it % NWS, ph = (it / NWS) & 1;
          mbar_wait(&wempty[s], ph ^ 1);
          mbar_arrive_expect_tx(&wfull[s], WST);
          tma_load_2d(sW + s * WST, &tmW, &wfull[s], (int32_t)(kc * BK), 0);
        }
      }
    }
  } else if (warp == W_XPROD) {
    if (lane == 0) {
      // the hi plane stays in L2 for the siblings' product 2 (evict_last); the lo plane is read once
      const uint64_t keep = policy_evict_last(), drop = policy_evict_first();
      // L2 prefetch cursor p.pf chunks ahead of the loads (bytes in flight beyond the 2 smem stages)
      int64_t prho = 0, pkc = 0;
      auto prefetch = [&]() {
        while (prho < nrounds && own_tile(prho) < 0) ++prho;
        if (prho >= nrounds) return;
        const int64_t t = own_tile(prho);
        tma_prefetch_2d(&tmX, (int32_t)(pkc * BK), (int32_t)(t * BM));
        if (LO) tma_prefetch_2d(&tmXlo, (int32_t)(pkc * BK), (int32_t)(t * BM));
        if (++pkc == p.nk) { pkc = 0; ++prho; }
      };
      for (int i = 0; i < p.pf; ++i) prefetch();
      uint32_t it = 0;
      for (int64_t rho = 0; rho < nrounds; ++rho) {
        const int64_t t = own_tile(rho);
        if (t < 0) continue;
        if (p.lag > 0)
          while (*bdone < rho - p.lag) __nanosleep(64);
        for (int64_t kc = 0; kc < p.nk; ++kc, ++it) {
          const uint32_t s = it % NSTA, ph = (it / NSTA) & 1;
          if (p.pf) prefetch();
          mbar_wait(&aempty[s], ph ^ 1);
          mbar_arrive_expect_tx(&afull[s], XSTG);
          if (p.hi_policy == 1)
            tma_load_2d(sA + s * XSTG, &tmX, &afull[s], (int32_t)(kc * BK), (int32_t)(t * BM));
          else
            tma_load_2d_hint(sA + s * XSTG, &tmX, &afull[s], (int32_t)(kc * BK), (int32_t)(t * BM),
                             p.hi_policy == 2 ? drop : keep);
          if (LO) tma_load_2d_hint(sA + s * XSTG + XPL, &tmXlo, &afull[s], (int32_t)(kc * BK), (int32_t)(t * BM), drop);
        }
      }
    }
  } else if (warp == W_BPROD) {
    if (lane == 0) {
      // B-stream: this thread loads the product-2 stages AND issues their MMAs (a second tcgen05 issuer,
      // so the A-stream's MMA thread never waits for L2 / sibling flags and the HBM stream keeps flowing)
      constexpr uint32_t ID_Z = idesc(FMT_BF16, FMT_BF16, 128, NB, 1, 1);    // Xᵀ and Y both MN-major
      const uint64_t drop = policy_evict_first();
      const int64_t nst_total = (te > tb && !(p.dbg & 1)) ? (te - tb) * (BM / KR) : 0;
      auto load = [&](int64_t q) {                // B stage q = (tile tb + q / (BM/KR), part q % (BM/KR))
        const int64_t t = tb + q / (BM / KR);
        const int h = (int)(q % (BM / KR));
        if (h == 0) {
          if (ld_acquire_gpu(p.flags + t) != p.epoch) {
            const uint64_t t0 = globaltimer_ns();
            while (ld_acquire_gpu(p.flags + t) != p.epoch) {
              __nanosleep(32);
              if (globaltimer_ns() - t0 > kFlagTimeoutNs) {
                atomicOr(p.err, DEV_TIMEOUT);
                break;
              }
            }
          }
          fence_proxy_async_global();             // Yᵀ was written by generic stores on another SM
        }
        const uint32_t s = q % NSTB, ph = (q / NSTB) & 1;
        const int32_t row = (int32_t)(t * BM + h * KR);
        mbar_wait(&bempty[s], ph ^ 1);
        mbar_arrive_expect_tx(&bfull[s], BX + BY);
        uint8_t* st = sB + s * (BX + BY);
        for (int bl = 0; bl < NC * 2; ++bl)
          tma_load_2d_hint(st + bl * BBLK, &tmXb, &bfull[s], (int32_t)(g * DG + bl * 64), row, drop);
        tma_load_2d(st + BX, &tmY, &bfull[s], 0, row);             // Y_hi features
        tma_load_2d(st + BX + BBLK, &tmY, &bfull[s], 64, row);     // Y_lo features
      };
      uint32_t ls = 0;                            // own tiles whose S was issued
      for (int64_t q = 0; q < NSTB && q < nst_total; ++q) load(q);
      for (int64_t q = 0; q < nst_total; ++q) {
        const uint32_t s = q % NSTB, ph = (q / NSTB) & 1;
        mbar_wait(&bfull[s], ph);
        tc_fence_after();
        if ((q + 1) % ((int64_t)(BM / KR) * p.ndg) == 0) *bdone = (int)((q + 1) / ((BM / KR) * p.ndg));
        const uint32_t xb = smem_u32(sB + s * (BX + BY)), yb = xb + BX;
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
          for (int kk = 0; kk < KR / 16; ++kk)
            mma_bf16(tmem + TZ + c * NB, smem_desc_sw128(xb + c * 2 * BBLK + kk * 2048, BBLK, 1024),
                     smem_desc_sw128(yb + kk * 2048, BBLK, 1024), ID_Z, (q != 0 || kk != 0) ? 1u : 0u);
        // S = YᵀY of an own tile from the same staged Y rows (M = N = 128 = [Y_hi | Y_lo], K = the stage's
        // rows), chained over the tile's 4 stages in row order (the sequence kernel A2 uses)
        const int64_t tq = q / (BM / KR);
        const int hq = (int)(q % (BM / KR));
        if ((tq % p.ndg) == g) {
          if (hq == 0) {
            mbar_wait(sempty, (ls & 1) ^ 1);
            tc_fence_after();
          }
#pragma unroll
          for (int kk = 0; kk < KR / 16; ++kk) {
            const uint64_t dy = smem_desc_sw128(yb + kk * 2048, BBLK, 1024);
            mma_bf16(tmem + TS, dy, dy, ID_Z, (hq != 0 || kk != 0) ? 1u : 0u);
          }
          if (hq == BM / KR - 1) {
            mma_commit(sfull);
            ++ls;
          }
        }
        mma_commit(&bempty[s]);
        // refill this slot as soon as its MMAs complete (measured faster than a non-blocking refill that
        // waits for the next pass round: the load then issues later and fewer stages are in flight)
        if (q + NSTB < nst_total) load(q + NSTB);
      }
      mma_commit(zfull);
    }
  } else if (warp == W_MMA) {
    if (lane == 0) {
      constexpr uint32_t ID = idesc(FMT_BF16, FMT_BF16, BM, NB, 0, 0);       // product 1
      constexpr uint32_t ID_HI = idesc(FMT_BF16, FMT_BF16, BM, MP, 0, 0);
      uint32_t ia = 0, lt = 0;
      for (int64_t rho = 0; rho < nrounds; ++rho) {
        // ---- A-work: product 1 of the own tile
        if (own_tile(rho) >= 0) {
          mbar_wait(tempty, (lt & 1) ^ 1);
          tc_fence_after();
          for (int64_t g0 = 0; g0 < p.nk; g0 += KSEG) {
            const int64_t g1 = min(p.nk, g0 + KSEG);
            // segments: accumulate in TMEM within a segment; the epilogue sums segments in fp32 RN
            // (here nseg must be 1: d ≤ KSEG·BK; the host only selects the fused kernel then)
            for (int64_t kc = g0; kc < g1; ++kc, ++ia) {
              const uint32_t s = ia % NSTA, ph = (ia / NSTA) & 1;
              const uint32_t ws = ia % NWS, wph = (ia / NWS) & 1;
              mbar_wait(&wfull[ws], wph);
              mbar_wait(&afull[s], ph);
              tc_fence_after();
              const uint32_t xa = smem_u32(sA + s * XSTG), wa = smem_u32(sW + ws * WST);
#pragma unroll
              for (int kk = 0; kk < BK / 16; ++kk) {
                mma_bf16(tmem + TY, smem_desc_sw128(xa + kk * 32, 16, 1024), smem_desc_sw128(wa + kk * 32, 16, 1024), ID,
                         (kc != g0) || kk != 0);
                if (LO)
                  mma_bf16(tmem + TY, smem_desc_sw128(xa + XPL + kk * 32, 16, 1024),
                           smem_desc_sw128(wa + kk * 32, 16, 1024), ID_HI, 1);
              }
              mma_commit(&aempty[s]);
              mma_commit(&wempty[ws]);
            }
          }
          mma_commit(tfull);
          ++lt;
        }
      }
    }
  } else {
    // ------------------------------------------------------------------ epilogue (128 threads = 128 rows)
    const int tid = threadIdx.x;
    const uint32_t tl = (uint32_t)(warp * 32) << 16;
    double* Sp = p.Spart + (int64_t)blockIdx.x * 2 * MP * MP;
    for (int e = tid; e < 2 * MP * MP; e += 128) Sp[e] = 0.0;
    asm volatile("bar.sync 1, 128;" ::: "memory");
    float sacc[MP];
#pragma unroll
    for (int j = 0; j < MP; ++j) sacc[j] = 0.f;
    int pending = 0;
    auto flush = [&]() {
      double* row = Sp + tid * MP;
#pragma unroll
      for (int j = 0; j < MP; ++j) {
        row[j] += (double)sacc[j];
        sacc[j] = 0.f;
      }
      pending = 0;
    };
    uint32_t lt = 0;
    for (int64_t rho = 0; rho < nrounds; ++rho) {
      const int64_t t = own_tile(rho);
      if (t < 0) continue;
      float y[MP];
      mbar_wait(tfull, lt & 1);
      tc_fence_after();
#pragma unroll
      for (int c0 = 0; c0 < MP; c0 += 8) {
        float v[8], w[8];
        tmem_ld8(tmem + tl + TY + c0, v);
        tmem_ld8(tmem + tl + TY + MP + c0, w);
#pragma unroll
        for (int j = 0; j < 8; ++j) y[c0 + j] = v[j] + w[j];
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty);
      // this tile's Y row as bf16 pairs [hi | lo] (256 contiguous bytes), then the tile's ready flag
      const int64_t grow = t * BM + tid;
      if (grow < p.nrow_pad) {
        uint4* dst = reinterpret_cast<uint4*>(p.Yrm + grow * NB);
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) {
          uint32_t h[4], l[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float a0 = y[ch * 8 + 2 * q], a1 = y[ch * 8 + 2 * q + 1];
            const __nv_bfloat162 hv = __floats2bfloat162_rn(a0, a1);
            const __nv_bfloat162 lv = __floats2bfloat162_rn(a0 - __low2float(hv), a1 - __high2float(hv));
            h[q] = *reinterpret_cast<const uint32_t*>(&hv);
            l[q] = *reinterpret_cast<const uint32_t*>(&lv);
          }
          dst[ch] = make_uint4(h[0], h[1], h[2], h[3]);
          dst[8 + ch] = make_uint4(l[0], l[1], l[2], l[3]);
        }
      }
      fence_proxy_async_global();
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (tid == 0) {
        __threadfence();
        st_release_gpu(p.flags + t, p.epoch);
      }
      // S of the previous own tile (its chain ran on the B-stream after the tile's flag)
      if (lt > 0) {
        mbar_wait(sfull, (lt - 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int c0 = 0; c0 < MP; c0 += 16) {
          float a[16], b2[16];
          tmem_ld16(tmem + tl + TS + c0, a);
          tmem_ld16(tmem + tl + TS + MP + c0, b2);
#pragma unroll
          for (int q = 0; q < 16; ++q) sacc[c0 + q] += a[q] + b2[q];
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(sempty);
        if (++pending == SFLUSH) flush();
      }
      ++lt;
    }
    if (lt > 0) {
      mbar_wait(sfull, (lt - 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int c0 = 0; c0 < MP; c0 += 16) {
        float a[16], b2[16];
        tmem_ld16(tmem + tl + TS + c0, a);
        tmem_ld16(tmem + tl + TS + MP + c0, b2);
#pragma unroll
        for (int q = 0; q < 16; ++q) sacc[c0 + q] += a[q] + b2[q];
      }
      ++pending;
    }
    if (pending) flush();
    // Zᵀ partial of (row group r, d-group g): thread = d within a 128-chunk; row = D_hi + D_lo
    mbar_wait(zfull, 0);
    tc_fence_after();
    for (int c = 0; c < NC; ++c) {
      const int64_t dd = (int64_t)g * DG + c * 128 + warp * 32 + lane;
      float* out = p.Zp + ((int64_t)r * (p.ndg * DG) + dd) * MP;
#pragma unroll 1
      for (int c0 = 0; c0 < MP; c0 += 16) {
        float v[16], w[16];
        tmem_ld16(tmem + tl + TZ + c * NB + c0, v);
        tmem_ld16(tmem + tl + TZ + c * NB + MP + c0, w);
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = nrounds == 0 ? 0.f : v[j] + w[j];
#pragma unroll
        for (int j = 0; j < 16; j += 4)
          *reinterpret_cast<float4*>(out + c0 + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == W_MMA) tmem_dealloc<512>(tmem);
}
