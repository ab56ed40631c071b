// tc_pair.cuh — the single-read power pass on d-sliced CTA pairs (§8 row a2; round 2): Y = X·W'ᵀ, S = YᵀY and
// Zᵀ = X_hiᵀ·Y (Y = Y_hi + Y_lo) with no X re-read from HBM and no Y round trip through global memory.
//
// A cluster of 2 CTAs owns a row group; both CTAs walk ALL the group's 128-row tiles, CTA h only the columns
// [h·SL, (h+1)·SL) of them (SL = 512, so d ≤ 1024):
//   product 1:  P_h = X[t, slice h]·W'[:, slice h]ᵀ                          (HBM stream of both planes)
//   exchange:   Y = P_0 + P_1 through distributed shared memory — rows [0, 64) are summed by rank 0, rows
//               [64, 128) by rank 1 (reduce-scatter), and each summed row, rounded to the bf16 pair
//               [Y_hi | Y_lo], is written into BOTH CTAs' Y slot (all-gather), already in the UMMA layout
//   product 2:  Zᵀ[slice h] += X_hi[t, slice h]ᵀ·Y_hi + X_hi[t, slice h]ᵀ·Y_lo   (the CTA's own slice of the
//               tile, re-read from L2 a few µs after its HBM read: the per-CTA working set is ~3 tiles)
//   S:          the tile's S = [Y_hi|Y_lo]ᵀ[Y_hi|Y_lo] chained on the tensor cores by rank (t mod 2).
// Compared with the row-group kernel (tc_fused.cuh) nothing crosses L2 but X itself, W' chunks and the
// CTA's own X_hi slice: no sibling re-reads of other CTAs' tiles, no Y rows in global memory, no flags.
// The only inter-CTA waits are inside a cluster (co-scheduled by construction), so no cooperative launch.
//
// TMEM (512 columns): Y partial [0, 128) (product 1, N = [W_hi; W_lo]), S [128, 256), Zᵀ [256, 512) = 4
// d-chunks of 128 rows × N = 64 (the Y_hi and Y_lo products accumulate into the same columns).
// Numerics: product 1 as kernel A2 (X_hi·[W_hi;W_lo]ᵀ + X_lo·W_hiᵀ) over ≤ 8 chunks per CTA, the two halves
// of the K range added in fp32 RN; product 2 reads X_hi with Y as the bf16 pair.
#pragma once

namespace kp2 {
constexpr int BM = 128, BK = 64, SFLUSH = 8;
constexpr int MP = 64, NB = 2 * MP;            // m padded; product-1 N ([W_hi; W_lo])
constexpr int SL = 512;                        // columns per CTA (d-slice)
constexpr int NCH = SL / BK;                   // 64-column chunks per slice
constexpr int MC = SL / 128;                   // 128-row d-chunks of Zᵀ per slice
constexpr uint32_t XPL = BM * 128;             // one bf16 plane chunk: 128 rows × 64 columns
constexpr uint32_t WST = NB * 128;             // W' chunk: 128 rows ([W_hi; W_lo]) × 64 columns
constexpr uint32_t YSL = 2 * BM * 128;         // Y slot: Y_hi block (128 rows × 128 B) + Y_lo block
constexpr uint32_t YLO = BM * 128;             // offset of the Y_lo block
constexpr int W_WPROD = 4, W_XPROD = 5, W_BPROD = 6, W_MMA = 7;
constexpr int NTHREADS = 8 * 32;
constexpr uint32_t TY = 0, TS = 128, TZ = 256;
}  // namespace kp2

struct KP2Params {
  int64_t n, d;
  int64_t ntiles;
  int nrg;
  int64_t tiles_per_rg;          // row group r: tiles [r·tpr, min(ntiles, (r+1)·tpr))
  double* Spart;                 // [grid][2·MP][MP]
  float* Zp;                     // [nrg][2·SL][MP]
  int pol;                       // L2 policies (policy_sel codes): A-stream hi | lo << 2 | product-2 re-read << 4
  long long* trace;              // experiment builds only: per-tile clock64 stamps of cluster 0 (nullptr: off)
};

// tools/ timeline of one cluster (experiment builds): trace[(h·KP2_TRACE_TILES + i)·KP2_TRACE_EV + e]
constexpr int KP2_TRACE_TILES = 128, KP2_TRACE_EV = 12;
#ifdef PPCA_EXPERIMENTS
#define KP2_STAMP(ev, i)                                                                                        \
  do {                                                                                                      \
    if (p.trace && r == 0 && (i) < KP2_TRACE_TILES)                                                         \
      p.trace[((int64_t)h * KP2_TRACE_TILES + (i)) * KP2_TRACE_EV + (ev)] = clock64();                      \
  } while (0)
#else
#define KP2_STAMP(ev, i) \
  do {                   \
  } while (0)
#endif

__device__ __forceinline__ uint32_t mapa_u32(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared::cluster.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}
// bulk copy of `bytes` from this CTA's shared memory to the peer's (dst, bar: shared::cluster addresses); the peer's
// mbarrier receives complete_tx
__device__ __forceinline__ void bulk_copy_to_peer(uint32_t dst, uint32_t src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "r"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async_cluster() {
  asm volatile("fence.proxy.async.shared::cluster;" ::: "memory");
}
// completion of this thread's earlier tcgen05 ops → one arrival on the barrier at bar's offset in every CTA of mask
__device__ __forceinline__ void mma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
               ::"r"(smem_u32(bar)), "h"(mask) : "memory");
}

template <int XM, int NSTA, int NWS, int NSTB, int KR>
__global__ void __launch_bounds__(kp2::NTHREADS, 1)
    xwz_pair_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                    const __grid_constant__ CUtensorMap tmXlo, const __grid_constant__ CUtensorMap tmXb,
                    KP2Params p) {
  pdl_wait();   // a programmatic dependent launch: inputs of the previous grid visible
  using namespace kp2;
  constexpr bool LO = XM == 2;
  constexpr uint32_t XSTG = LO ? 2 * XPL : XPL;
  constexpr uint32_t BBLK = KR * 128;            // one 64-column block of a B stage (KR rows)
  constexpr uint32_t BSTG = NCH * BBLK;          // B stage: KR rows × SL columns of X_hi
  constexpr int BPT = BM / KR;                   // B stages per tile
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = sm;                               // NSTA × XSTG
  uint8_t* sW = sA + NSTA * XSTG;                 // NWS × WST
  uint8_t* sB = sW + NWS * WST;                   // NSTB × BSTG
  uint8_t* sY = sB + NSTB * BSTG;                 // 2 × YSL (Y slots of tiles i even / odd)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sY + 2 * YSL);
  uint64_t* afull = bars;                         // NSTA
  uint64_t* aempty = afull + NSTA;
  uint64_t* wfull = aempty + NSTA;                // NWS
  uint64_t* wempty = wfull + NWS;
  uint64_t* bfull = wempty + NWS;                 // NSTB
  uint64_t* bempty = bfull + NSTB;
  uint64_t* tfull = bempty + NSTB;                // Y partial accumulated / drained
  uint64_t* tempty = tfull + 1;
  uint64_t* sempty = tempty + 1;
  uint64_t* sfull = sempty + 1;
  uint64_t* zfull = sfull + 1;
  uint64_t* rsfull = zfull + 1;                   // [2] the peer's partial rows landed in the slot (bulk copy, 16 KB)
  uint64_t* yfull = rsfull + 2;                   // [2] all 128 Y rows in the slot (own rows + the peer's bulk copy)
  uint64_t* yempty = yfull + 2;                   // [2] both CTAs' product 2 of the slot's last tile done (2)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(yempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t h = pair_rank(), peer = h ^ 1u;
  const int r = blockIdx.x >> 1;
  const int64_t tb = (int64_t)r * p.tiles_per_rg, te = min(p.ntiles, tb + p.tiles_per_rg);
  const int64_t ntl = te > tb ? te - tb : 0;     // tiles of this row group
  const int64_t c0 = (int64_t)h * SL;            // first column of the slice
  const int64_t len = min((int64_t)SL, p.d - c0);
  const int nk = (int)((len + BK - 1) / BK);     // 64-column chunks of the slice
  const int mc = (int)((len + 127) / 128);       // 128-column d-chunks of Zᵀ

  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTA; ++s) { mbar_init(&afull[s], 1); mbar_init(&aempty[s], 1); }
    for (int s = 0; s < NWS; ++s) { mbar_init(&wfull[s], 1); mbar_init(&wempty[s], 1); }
    for (int s = 0; s < NSTB; ++s) { mbar_init(&bfull[s], 1); mbar_init(&bempty[s], 1); }
    mbar_init(tfull, 1);
    mbar_init(tempty, 4);
    mbar_init(sempty, 4);
    mbar_init(sfull, 1);
    mbar_init(zfull, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&rsfull[s], 1);                   // own-row leader's expect_tx + the peer's bulk copy
      mbar_init(&yfull[s], 1);                    // own-row leader's expect_tx + the peer's bulk copy
      mbar_init(&yempty[s], 2);
    }
    fence_barrier_init();
  }
  if (warp == W_XPROD && lane == 0) {
    tma_prefetch_desc(&tmW);
    tma_prefetch_desc(&tmX);
    if (LO) tma_prefetch_desc(&tmXlo);
    tma_prefetch_desc(&tmXb);
  }
  if (warp == W_MMA) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  cluster_barrier();                              // the peer's barriers exist before any remote arrive
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == W_WPROD) {
    if (lane == 0) {
      // the L2 producer: W' chunks (product 1) and the X_hi slice stages of product 2, polled round-robin so
      // that neither ring waits behind the other (both are L2 hits; W' first: it gates the HBM stream)
      const uint64_t drop = policy_sel((p.pol >> 4) & 3);
      const int nbl = 2 * mc;
      const int64_t nw = ntl * nk, nq = ntl * BPT;
      int64_t iw = 0, q = 0;
      while (iw < nw || q < nq) {
        if (iw < nw) {
          const uint32_t s = iw % NWS, ph = (iw / NWS) & 1;
          if (mbar_test(&wempty[s], ph ^ 1)) {
            mbar_arrive_expect_tx(&wfull[s], WST);
            tma_load_2d(sW + s * WST, &tmW, &wfull[s], (int32_t)(c0 + (iw % nk) * BK), 0);
            ++iw;
          }
        }
        if (q < nq) {
          const uint32_t s = q % NSTB, ph = (q / NSTB) & 1;
          if (mbar_test(&bempty[s], ph ^ 1)) {
            const int64_t t = tb + q / BPT;
            const int hq = (int)(q % BPT);
            mbar_arrive_expect_tx(&bfull[s], nbl * BBLK);
            uint8_t* st = sB + s * BSTG;
            for (int bl = 0; bl < nbl; ++bl)
              tma_load_2d_hint(st + bl * BBLK, &tmXb, &bfull[s], (int32_t)(c0 + bl * 64), (int32_t)(t * BM + hq * KR),
                               drop);
            ++q;
          }
        }
      }
    }
  } else if (warp == W_XPROD) {
    if (lane == 0) {
      // the hi plane is re-read by this CTA's product 2 a few µs later (evict_last); the lo plane is read once
      const uint64_t keep = policy_sel(p.pol & 3), drop = policy_sel((p.pol >> 2) & 3);
      uint32_t it = 0;
      for (int64_t i = 0; i < ntl; ++i) {
        const int64_t t = tb + i;
        for (int kc = 0; kc < nk; ++kc, ++it) {
          const uint32_t s = it % NSTA, ph = (it / NSTA) & 1;
          mbar_wait(&aempty[s], ph ^ 1);
          if (kc == 0) KP2_STAMP(8, i);
          if (kc == nk - 1) KP2_STAMP(9, i);
          mbar_arrive_expect_tx(&afull[s], XSTG);
          tma_load_2d_hint(sA + s * XSTG, &tmX, &afull[s], (int32_t)(c0 + kc * BK), (int32_t)(t * BM), keep);
          if (LO) tma_load_2d_hint(sA + s * XSTG + XPL, &tmXlo, &afull[s], (int32_t)(c0 + kc * BK), (int32_t)(t * BM), drop);
        }
      }
    }
  } else if (warp == W_BPROD) {
    if (lane == 0) {
      // product 2 (+ S): issues the MMAs of the CTA's X_hi slice stages (loaded by the L2 producer) once Y landed
      constexpr uint32_t ID_Z = idesc(FMT_BF16, FMT_BF16, 128, MP, 1, 1);    // Xᵀ and Y both MN-major
      constexpr uint32_t ID_S = idesc(FMT_BF16, FMT_BF16, 128, NB, 1, 1);    // [Y_hi|Y_lo]ᵀ[Y_hi|Y_lo]
      const int64_t nst_total = ntl * BPT;
      const uint32_t ys0 = smem_u32(sY);
      uint32_t ls = 0;
      for (int64_t q = 0; q < nst_total; ++q) {
        const int64_t i = q / BPT;
        const int hq = (int)(q % BPT);
        const uint32_t s = q % NSTB, ph = (q / NSTB) & 1;
        const uint32_t ysl = (uint32_t)(i & 1), yph = (uint32_t)(i >> 1) & 1;
        const uint32_t yb = ys0 + ysl * YSL;
        if (hq == 0) {
          mbar_wait_cluster(&yfull[ysl], yph);          // both CTAs' rows of Y(t) are in the slot
          KP2_STAMP(6, i);
        }
        mbar_wait(&bfull[s], ph);
        tc_fence_after();
        const uint32_t xb = smem_u32(sB + s * BSTG);
#pragma unroll 1
        for (int c = 0; c < mc; ++c)
#pragma unroll
          for (int kk = 0; kk < KR / 16; ++kk) {
            const uint64_t da = smem_desc_sw128(xb + c * 2 * BBLK + kk * 2048, BBLK, 1024);
            const uint32_t yrow = (uint32_t)(hq * KR + kk * 16) * 128u;
            mma_bf16(tmem + TZ + c * MP, da, smem_desc_sw128(yb + yrow, YLO, 1024), ID_Z, (q != 0 || kk != 0) ? 1u : 0u);
            mma_bf16(tmem + TZ + c * MP, da, smem_desc_sw128(yb + YLO + yrow, YLO, 1024), ID_Z, 1u);
          }
        mma_commit(&bempty[s]);
        if (hq == BPT - 1) {
          if ((uint32_t)((tb + i) & 1) == h) {        // this CTA forms the tile's S from the same Y slot
            mbar_wait(sempty, (ls & 1) ^ 1);
            tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < BM / 16; ++kk) {
              const uint64_t dy = smem_desc_sw128(yb + kk * 2048, YLO, 1024);
              mma_bf16(tmem + TS, dy, dy, ID_S, kk != 0 ? 1u : 0u);
            }
            mma_commit(sfull);
            ++ls;
          }
          KP2_STAMP(7, i);
          mma_commit_mc(&yempty[ysl], 3);             // this CTA no longer reads the slot (both CTAs count it)
        }
      }
      mma_commit(zfull);
    }
  } else if (warp == W_MMA) {
    if (lane == 0) {
      constexpr uint32_t ID = idesc(FMT_BF16, FMT_BF16, BM, NB, 0, 0);       // product 1
      constexpr uint32_t ID_HI = idesc(FMT_BF16, FMT_BF16, BM, MP, 0, 0);
      uint32_t ia = 0;
#ifdef PPCA_EXPERIMENTS
      auto gstamp = [&](int k) {                      // wall clock of every CTA: start / end of product 1
        if (p.trace) {
          uint64_t g;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
          p.trace[2 * KP2_TRACE_TILES * KP2_TRACE_EV + 2 * blockIdx.x + k] = (long long)g;
        }
      };
      gstamp(0);
#endif
      for (int64_t i = 0; i < ntl; ++i) {
        mbar_wait(tempty, ((uint32_t)i & 1) ^ 1);
        tc_fence_after();
        KP2_STAMP(0, i);
#ifdef PPCA_EXPERIMENTS
        if (p.trace && r == 0 && i < KP2_TRACE_TILES) {   // SM clock vs wall clock
          uint64_t g;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
          p.trace[((int64_t)h * KP2_TRACE_TILES + i) * KP2_TRACE_EV + 10] = (long long)g;
        }
#endif
        for (int kc = 0; kc < nk; ++kc, ++ia) {
          const uint32_t s = ia % NSTA, ph = (ia / NSTA) & 1;
          const uint32_t ws = ia % NWS, wph = (ia / NWS) & 1;
          mbar_wait(&wfull[ws], wph);
          mbar_wait(&afull[s], ph);
          tc_fence_after();
          const uint32_t xa = smem_u32(sA + s * XSTG), wa = smem_u32(sW + ws * WST);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            mma_bf16(tmem + TY, smem_desc_sw128(xa + kk * 32, 16, 1024), smem_desc_sw128(wa + kk * 32, 16, 1024), ID,
                     (kc != 0 || kk != 0) ? 1u : 0u);
            if (LO)
              mma_bf16(tmem + TY, smem_desc_sw128(xa + XPL + kk * 32, 16, 1024), smem_desc_sw128(wa + kk * 32, 16, 1024),
                       ID_HI, 1u);
          }
          mma_commit(&aempty[s]);
          mma_commit(&wempty[ws]);
        }
        KP2_STAMP(1, i);
        mma_commit(tfull);
      }
#ifdef PPCA_EXPERIMENTS
      gstamp(1);
#endif
    }
  } else {
    // ------------------------------------------------------------------ epilogue (128 threads = 128 tile rows)
    const int tid = threadIdx.x;
    const uint32_t tl = (uint32_t)(warp * 32) << 16;
    const bool own = (uint32_t)(warp >> 1) == h;      // rows [64h, 64h + 64) are summed here
    // Y slot rows in the UMMA SW128 MN-major layout: row r = 128 B in the Y_hi block + 128 B in the Y_lo block,
    // 16-byte chunk q at position q ^ (r & 7).  The peer's reduce-scatter rows (fp32, 64 values = 256 B) land in
    // exactly the bytes of the receiving thread's own Y row, which that thread overwrites with the bf16 pair.
    const uint32_t row = (uint32_t)tid;
    const uint32_t rbase = (row >> 3) * 1024u + (row & 7u) * 128u;
    auto chunk_off = [&](int q) -> uint32_t {       // 16-byte chunk q (0..15) of row `row`: [hi block | lo block]
      return (q < 8 ? 0u : YLO) + rbase + ((((uint32_t)q & 7u) ^ (row & 7u)) << 4);
    };
    const uint32_t sY_u = smem_u32(sY), sY_peer = mapa_u32(sY_u, peer);
    const uint32_t rsfull_peer = mapa_u32(smem_u32(rsfull), peer), yfull_peer = mapa_u32(smem_u32(yfull), peer);
    double* Sp = p.Spart + (int64_t)blockIdx.x * 2 * MP * MP;
    for (int e = tid; e < 2 * MP * MP; e += 128) Sp[e] = 0.0;
    asm volatile("bar.sync 1, 128;" ::: "memory");
    float sacc[MP];
#pragma unroll
    for (int j = 0; j < MP; ++j) sacc[j] = 0.f;
    int pending = 0;
    uint32_t ls = 0;
    auto drain_s = [&]() {                             // S of an own tile: rows tid of the 128×128 chain
      mbar_wait(sfull, ls & 1);
      tc_fence_after();
#pragma unroll
      for (int cc = 0; cc < MP; cc += 16) {
        float a[16], b2[16];
        tmem_ld16(tmem + tl + TS + cc, a);
        tmem_ld16(tmem + tl + TS + MP + cc, b2);
#pragma unroll
        for (int q = 0; q < 16; ++q) sacc[cc + q] += a[q] + b2[q];
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(sempty);
      ++ls;
      if (++pending == SFLUSH) {
        double* srow = Sp + tid * MP;
#pragma unroll
        for (int j = 0; j < MP; ++j) {
          srow[j] += (double)sacc[j];
          sacc[j] = 0.f;
        }
        pending = 0;
      }
    };
    for (int64_t i = 0; i < ntl; ++i) {
      const int64_t t = tb + i;
      float y[MP];
      mbar_wait(tfull, (uint32_t)i & 1);
      tc_fence_after();
      if (lane == 0 && (warp & 1) == 0) KP2_STAMP(2 + warp, i);
#pragma unroll
      for (int cc = 0; cc < MP; cc += 8) {
        float v[8], w[8];
        tmem_ld8(tmem + tl + TY + cc, v);
        tmem_ld8(tmem + tl + TY + MP + cc, w);
#pragma unroll
        for (int j = 0; j < 8; ++j) y[cc + j] = v[j] + w[j];
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty);
      const uint32_t ysl = (uint32_t)(i & 1), yph = (uint32_t)(i >> 1) & 1;
      const uint32_t so = ysl * YSL;
      // the slot's previous tile (i − 2) is done in both CTAs' product 2
      if (i >= 2) mbar_wait_cluster(&yempty[ysl], yph ^ 1);
      // the 64-row half of a slot owned by rank x: rows [64x, 64x + 64) of the Y_hi block and of the Y_lo block
      const uint32_t half_peer = so + (uint32_t)peer * 8192u, half_own = so + h * 8192u;
      if (!own) {
        // reduce-scatter: the partial rows staged in this CTA's slot at the peer's own-row bytes, then one bulk
        // copy per block to the same bytes of the peer's slot (complete_tx on the peer's rsfull)
#pragma unroll
        for (int q = 0; q < 16; ++q)
          *reinterpret_cast<float4*>(sY + so + chunk_off(q)) = make_float4(y[4 * q], y[4 * q + 1], y[4 * q + 2], y[4 * q + 3]);
        fence_proxy_async_smem();
        asm volatile("bar.sync %0, 64;" ::"r"(2 + (int)peer) : "memory");
        if (tid == 64 * (int)peer) {
          bulk_copy_to_peer(sY_peer + half_peer, sY_u + half_peer, 8192u, rsfull_peer + ysl * 8u);
          bulk_copy_to_peer(sY_peer + YLO + half_peer, sY_u + YLO + half_peer, 8192u, rsfull_peer + ysl * 8u);
        }
      } else {
        if (tid == 64 * (int)h) mbar_arrive_expect_tx(&rsfull[ysl], 16384u);
        mbar_wait_cluster(&rsfull[ysl], yph);
        float pp[MP];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const float4 v = *reinterpret_cast<const float4*>(sY + so + chunk_off(q));
          pp[4 * q] = v.x; pp[4 * q + 1] = v.y; pp[4 * q + 2] = v.z; pp[4 * q + 3] = v.w;
        }
        // Y = P_0 + P_1 (fp32 RN), the bf16 pair into this CTA's slot, then one bulk copy per block to the peer
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) {
          uint32_t hw[4], lw[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float a0 = y[ch * 8 + 2 * q] + pp[ch * 8 + 2 * q], a1 = y[ch * 8 + 2 * q + 1] + pp[ch * 8 + 2 * q + 1];
            const __nv_bfloat162 hv = __floats2bfloat162_rn(a0, a1);
            const __nv_bfloat162 lv = __floats2bfloat162_rn(a0 - __low2float(hv), a1 - __high2float(hv));
            hw[q] = *reinterpret_cast<const uint32_t*>(&hv);
            lw[q] = *reinterpret_cast<const uint32_t*>(&lv);
          }
          const uint32_t off = so + rbase + ((((uint32_t)ch) ^ (row & 7u)) << 4);
          *reinterpret_cast<uint4*>(sY + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
          *reinterpret_cast<uint4*>(sY + YLO + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
        }
        fence_proxy_async_smem();                      // generic writes → the bulk copy and both tensor cores
        asm volatile("bar.sync %0, 64;" ::"r"(2 + (int)h) : "memory");
        if (tid == 64 * (int)h) {
          bulk_copy_to_peer(sY_peer + half_own, sY_u + half_own, 8192u, yfull_peer + ysl * 8u);
          bulk_copy_to_peer(sY_peer + YLO + half_own, sY_u + YLO + half_own, 8192u, yfull_peer + ysl * 8u);
          mbar_arrive_expect_tx(&yfull[ysl], 16384u);  // own rows written; the peer's 16 KB arrive by its copy
        }
      }
      if (lane == 0 && (warp & 1) == 0) KP2_STAMP(3 + warp, i);
      // S of the previous tile, if this CTA chained it
      if (i > 0 && (uint32_t)((t - 1) & 1) == h) drain_s();
    }
    if (ntl > 0 && (uint32_t)((te - 1) & 1) == h) drain_s();
    if (pending) {
      double* row = Sp + tid * MP;
#pragma unroll
      for (int j = 0; j < MP; ++j) row[j] += (double)sacc[j];
    }
    // Zᵀ partial of (row group r, slice h): thread = d within a 128-chunk
    mbar_wait(zfull, 0);
    tc_fence_after();
    for (int c = 0; c < mc; ++c) {
      const int64_t dd = c0 + c * 128 + warp * 32 + lane;
      float* out = p.Zp + ((int64_t)r * (2 * SL) + dd) * MP;
#pragma unroll 1
      for (int cc = 0; cc < MP; cc += 16) {
        float v[16];
        tmem_ld16(tmem + tl + TZ + c * MP + cc, v);
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = ntl == 0 ? 0.f : v[j];
#pragma unroll
        for (int j = 0; j < 16; j += 4)
          *reinterpret_cast<float4*>(out + cc + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_barrier();                                  // no remote store / arrive may target an exited CTA
  if (warp == W_MMA) tmem_dealloc<512>(tmem);
}
