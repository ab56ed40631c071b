// tc_xty.cuh — kernel B of the tensor-core pass:  Zᵀ[d-chunk] += X_tᵀ·Y_t   (§8 row a2, product 2).
//
// Work item = (d-group of NC×128 columns, row group).  A = X_tᵀ (M = 128 d-values, K = rows) is the
// staged X tile read MN-major; B = [Y_hi; Y_lo]ᵀ (N = 2·MP, K = rows) comes from the bf16-pair Yᵀ
// written by kernel A, so Z = X_hiᵀ(Y_hi + Y_lo) keeps Y to ~2^-17 (a single bf16 Y moves the next
// iterate's span at first order — 1.5e-4 on the Ritz values of C3s, measured against the oracle).
// The partial Zᵀ of an item stays in TMEM over its rows and is written once; a fixed-order
// reduction over row groups produces Z.
#pragma once

namespace kb {
constexpr int KR = 64;          // rows (K) per stage
constexpr int NST = 4;
constexpr int NCONV = 8;
constexpr int PF = 0;           // converter L2-prefetch distance in half-stages (measured: hurts; off)
constexpr int W_CONV0 = 4, W_PROD = 12, W_MMA = 13;
constexpr int NTHREADS = 14 * 32;
constexpr uint32_t BLK = KR * 128;            // one 64-column block of a stage (bytes)
// XLO: the X_lo plane of a split X is staged too and X_loᵀ·Y_hi is added (the minibatch steps, whose
// products are the update itself; the power pass reads X_hi only)
template <int MP, bool XLO = false, bool LEAN = false> struct Cfg {
  // 256-column d-groups for every m: the Yᵀ operand (2·MP rows per 64-row stage) is then streamed from L2 once
  // per 256 X columns (C5, MP = 128: with 128-column groups Yᵀ moved twice X's bytes through L2)
  static constexpr int NC = 2;                            // 128-wide d chunks per work item
  static constexpr int NB = LEAN ? MP : 2 * MP;          // UMMA N: [Y_hi; Y_lo] (Y_hi alone: bf16 X, R27)
  static constexpr uint32_t XST = NC * 2 * BLK;          // X stage bytes (one plane)
  static constexpr uint32_t XSTG = XLO ? 2 * XST : XST;  // X stage bytes (all planes)
  static constexpr uint32_t YST = NB * 128;              // Yᵀ stage bytes (NB rows × 64 K)
  static constexpr uint32_t ACC = NC * NB;               // TMEM columns per accumulator buffer
  static constexpr int NBUF = 2 * ACC <= 512 ? 2 : 1;     // double-buffered items when they fit in TMEM
  static constexpr uint32_t TCOLS = NBUF * ACC <= 64 ? 64 : (NBUF * ACC <= 128 ? 128 : (NBUF * ACC <= 256 ? 256 : 512));
  static constexpr int NSTFIT = (int)((227 * 1024 - 1280) / (XSTG + YST));
  static constexpr int NSTG = NSTFIT < NST ? NSTFIT : NST;
  static constexpr size_t SMEM = 1024 + NSTG * (XSTG + YST) + 256;
};
}  // namespace kb

struct KBParams {
  const void* X;
  int64_t n, d, ld;
  int m, mp;
  int64_t ndg;              // d-groups (NC × 128 columns each)
  int64_t nrg;              // row groups
  int64_t rows_per_rg;      // multiple of KR
  float* Zp;                // [nrg][d_pad][mp] fp32 partials (d_pad = ndg·NC·128)
};

template <int MP, bool XBF16, bool XLO = false, bool LEAN = false>
__global__ void __launch_bounds__(kb::NTHREADS, 1)
    xty_tc_kernel(const __grid_constant__ CUtensorMap tmYT, const __grid_constant__ CUtensorMap tmX,
                  const __grid_constant__ CUtensorMap tmXlo, KBParams p) {
  pdl_wait();   // a programmatic dependent launch: inputs of the previous grid visible
  using namespace kb;
  using CF = Cfg<MP, XLO, LEAN>;
  constexpr int NC = CF::NC, NB = CF::NB, NST = CF::NSTG, NBUF = CF::NBUF;
  constexpr uint32_t XST = CF::XSTG, XPL = CF::XST, YST = CF::YST, ACC = CF::ACC, TCOLS = CF::TCOLS;
  static_assert(!XLO || XBF16, "the X_lo plane is staged by TMA");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sX = sm;
  uint8_t* sY = sX + NST * XST;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sY + NST * YST);
  uint64_t* full = bars;
  uint64_t* empty = bars + NST;
  uint64_t* tfull = bars + 2 * NST;
  uint64_t* tempty = bars + 2 * NST + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * NST + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], XBF16 ? 1 : NCONV + 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
    }
    fence_barrier_init();
  }
  if (warp == W_PROD && lane == 0) {
    tma_prefetch_desc(&tmYT);
    if (XBF16) tma_prefetch_desc(&tmX);
    if (XLO) tma_prefetch_desc(&tmXlo);
  }
  if (warp == W_MMA) tmem_alloc<TCOLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int64_t nitems = p.ndg * p.nrg;
  auto item_rows = [&](int64_t item, int64_t& r0, int64_t& nks) {
    const int64_t rg = item / p.ndg;      // CTAs working concurrently share a row group: Yᵀ hits L2
    r0 = rg * p.rows_per_rg;
    const int64_t r1 = min(p.n, r0 + p.rows_per_rg);
    nks = r1 > r0 ? (r1 - r0 + KR - 1) / KR : 0;
  };

  if (warp == W_PROD) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      uint32_t it = 0;
      for (int64_t item = blockIdx.x; item < nitems; item += gridDim.x) {
        int64_t r0, nks;
        item_rows(item, r0, nks);
        const int64_t c0 = (item % p.ndg) * (NC * 128);
        for (int64_t ks = 0; ks < nks; ++ks, ++it) {
          const uint32_t s = it % NST, ph = (it / NST) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          mbar_arrive_expect_tx(&full[s], YST + (XBF16 ? XST : 0));
          tma_load_2d(sY + s * YST, &tmYT, &full[s], (int32_t)(r0 + ks * KR), 0);
          if (XBF16)
            for (int bl = 0; bl < NC * 2; ++bl)
              tma_load_2d_hint(sX + s * XST + bl * BLK, &tmX, &full[s], (int32_t)(c0 + bl * 64),
                               (int32_t)(r0 + ks * KR), pol);
          if (XLO)
            for (int bl = 0; bl < NC * 2; ++bl)
              tma_load_2d_hint(sX + s * XST + XPL + bl * BLK, &tmXlo, &full[s], (int32_t)(c0 + bl * 64),
                               (int32_t)(r0 + ks * KR), pol);
        }
      }
    }
  } else if (warp == W_MMA) {
    constexpr uint32_t ID = idesc(FMT_BF16, FMT_BF16, 128, NB, 1, 0);    // A = Xᵀ MN-major, B = Yᵀ K-major
    constexpr uint32_t ID_HI = idesc(FMT_BF16, FMT_BF16, 128, MP, 1, 0);  // X_loᵀ·Y_hi into the hi columns
    uint32_t it = 0, tt = 0;
    for (int64_t item = blockIdx.x; item < nitems; item += gridDim.x, ++tt) {
      int64_t r0, nks;
      item_rows(item, r0, nks);
      const uint32_t b = NBUF == 2 ? (tt & 1) : 0, tph = NBUF == 2 ? ((tt >> 1) & 1) : (tt & 1);
      mbar_wait(&tempty[b], tph ^ 1);
      tc_fence_after();
      for (int64_t ks = 0; ks < nks; ++ks, ++it) {
        const uint32_t s = it % NST, ph = (it / NST) & 1;
        mbar_wait(&full[s], ph);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t xa = smem_u32(sX + s * XST), ya = smem_u32(sY + s * YST);
#pragma unroll
          for (int c = 0; c < NC; ++c)
#pragma unroll
            for (int kk = 0; kk < KR / 16; ++kk)
            {
              mma_bf16(tmem + b * ACC + c * NB, smem_desc_sw128(xa + c * 2 * BLK + kk * 2048, BLK, 1024),
                       smem_desc_sw128(ya + kk * 32, 16, 1024), ID, (ks | kk) != 0);
              if (XLO)
                mma_bf16(tmem + b * ACC + c * NB, smem_desc_sw128(xa + XPL + c * 2 * BLK + kk * 2048, BLK, 1024),
                         smem_desc_sw128(ya + kk * 32, 16, 1024), ID_HI, 1);
            }
          mma_commit(&empty[s]);
        }
        __syncwarp();
      }
      if (lane == 0) mma_commit(&tfull[b]);
      __syncwarp();
    }
  } else if (warp >= W_CONV0 && warp < W_CONV0 + NCONV) {
    if (!XBF16) {
      // A stage = KR rows × NC·128 fp32 columns, converted in two half-stages of KR/2 rows; each warp
      // instruction covers one row × 128 columns (512 B).  Half-stages are double-buffered in
      // registers so one is in flight while the other is stored.
      const float* X = reinterpret_cast<const float*>(p.X);
      const int cw = warp - W_CONV0;
      constexpr int PER = (KR / 2) * NC * 128 / 4 / (NCONV * 32);   // float4 per thread per half-stage
      // flatten (item, stage, half) into a sequence index
      int64_t my_items = 0;
      for (int64_t item = blockIdx.x; item < nitems; item += gridDim.x) ++my_items;
      struct Pos { int64_t item, ks, nks, r0; int h; uint32_t it; };
      // iterator over this CTA's half-stages
      int64_t cur_item = blockIdx.x, cur_ks = 0, cur_r0 = 0, cur_nks = 0;
      int cur_h = 0;
      uint32_t cur_it = 0;
      item_rows(cur_item, cur_r0, cur_nks);
      auto skip_empty = [&]() {
        while (cur_item < nitems && cur_ks >= cur_nks) {
          cur_item += gridDim.x;
          cur_ks = 0;
          if (cur_item < nitems) item_rows(cur_item, cur_r0, cur_nks);
        }
      };
      skip_empty();
      auto next_pos = [&](Pos& q) -> bool {
        if (cur_item >= nitems) return false;
        q.item = cur_item; q.ks = cur_ks; q.nks = cur_nks; q.r0 = cur_r0; q.h = cur_h; q.it = cur_it;
        if (++cur_h == 2) {
          cur_h = 0;
          ++cur_ks;
          ++cur_it;
          skip_empty();
        }
        return true;
      };
      // L2 prefetch PF half-stages ahead (a second cursor over the same sequence; one prefetch per line)
      int64_t pf_item = cur_item, pf_ks = 0, pf_r0 = cur_r0, pf_nks = cur_nks;
      int pf_h = 0;
      auto prefetch_next = [&]() {
        while (pf_item < nitems && pf_ks >= pf_nks) {
          pf_item += gridDim.x;
          pf_ks = 0;
          if (pf_item < nitems) item_rows(pf_item, pf_r0, pf_nks);
        }
        if (pf_item >= nitems) return;
        const int64_t c0 = (pf_item % p.ndg) * (NC * 128);
#pragma unroll
        for (int i = 0; i < PER; ++i) {
          const int f = (i * NCONV + cw) * 32 + lane;
          const int row = f / (NC * 32), c4 = f % (NC * 32);
          const int64_t r = pf_r0 + pf_ks * KR + pf_h * (KR / 2) + row, col = c0 + c4 * 4;
          if ((c4 & 7) == 0 && r < p.n && col < p.d) prefetch_l2(X + r * p.ld + col);
        }
        if (++pf_h == 2) { pf_h = 0; ++pf_ks; }
      };
      for (int i = 0; i < PF; ++i) prefetch_next();
      auto load = [&](const Pos& q, float4 (&r)[PER]) {
        if (PF) prefetch_next();
        const int64_t c0 = (q.item % p.ndg) * (NC * 128);
#pragma unroll
        for (int i = 0; i < PER; ++i) {
          const int f = (i * NCONV + cw) * 32 + lane;             // float4 index within the half-stage
          const int row = f / (NC * 32), c4 = f % (NC * 32);
          r[i] = ldg_x4(X, p.ld, q.r0 + q.ks * KR + q.h * (KR / 2) + row, p.n, c0 + c4 * 4, p.d);
        }
      };
      auto store = [&](const Pos& q, const float4 (&r)[PER]) {
        const uint32_t s = q.it % NST, ph = (q.it / NST) & 1;
        if (q.h == 0) mbar_wait(&empty[s], ph ^ 1);
        uint8_t* st = sX + s * XST;
#pragma unroll
        for (int i = 0; i < PER; ++i) {
          const int f = (i * NCONV + cw) * 32 + lane;
          const int row = q.h * (KR / 2) + f / (NC * 32), col = (f % (NC * 32)) * 4;
          *reinterpret_cast<uint2*>(st + (col >> 6) * BLK + sw128(row, (col & 63) * 2)) = pack4_bf16(r[i]);
        }
        if (q.h == 1) {
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(&full[s]);
        }
      };
      (void)my_items;
      float4 A[PER], B[PER];
      Pos qa, qb;
      bool ha = next_pos(qa);
      if (ha) load(qa, A);
      while (ha) {
        const bool hb = next_pos(qb);
        if (hb) load(qb, B);
        store(qa, A);
        if (!hb) break;
        ha = next_pos(qa);
        if (ha) load(qa, A);
        store(qb, B);
      }
    }
  } else if (warp < 4) {
    // epilogue: thread = TMEM lane = d within a 128-chunk; Zᵀ row = D_hi + D_lo over m columns
    uint32_t tt = 0;
    for (int64_t item = blockIdx.x; item < nitems; item += gridDim.x, ++tt) {
      int64_t r0, nks;
      item_rows(item, r0, nks);
      const int64_t dg = item % p.ndg, rg = item / p.ndg;
      const uint32_t b = NBUF == 2 ? (tt & 1) : 0, tph = NBUF == 2 ? ((tt >> 1) & 1) : (tt & 1);
      mbar_wait(&tfull[b], tph);
      tc_fence_after();
      for (int c = 0; c < NC; ++c) {
        const int64_t dd = dg * NC * 128 + c * 128 + warp * 32 + lane;
        float* out = p.Zp + (rg * (p.ndg * NC * 128) + dd) * MP;
#pragma unroll 1
        for (int c0 = 0; c0 < MP; c0 += 16) {
          float v[16], w[16];
          const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + b * ACC + c * NB + c0;
          tmem_ld16(ta, v);
          if (!LEAN) tmem_ld16(ta + MP, w);
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = nks == 0 ? 0.f : (LEAN ? v[j] : v[j] + w[j]);
#pragma unroll
          for (int j = 0; j < 16; j += 4)
            *reinterpret_cast<float4*>(out + c0 + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[b]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == W_MMA) tmem_dealloc<TCOLS>(tmem);
}
