// tc_xw.cuh — kernel A of the tensor-core pass:  Y_t = X_t·W'ᵀ and S += Y_tᵀY_t   (§8 rows a2 / a7).
//
// Persistent, one CTA per SM, 128-row tiles (UMMA M = 128), 64-column K chunks (one 128-byte swizzle row).
// Warp roles (22 warps): 0–3 epilogue (TMEM lane quadrants), 4–19 converters (fp32 X → bf16 hi/lo, 8 rows
// each; 16 warps × 3 register buffers keep ~64 KB of loads in flight per SM), 20 W' TMA ring, 21 MMA issue
// (owns TMEM).  This kernel serves the plain fp32 layout; TMA-staged X runs kernel A2 (tc_xw2.cuh).
//
// Precision (measured, profiles/r1_tc_microtest.txt, tests/tc_accum_test.cu):
//  * kind::tf32 truncates fp32 operands  → operands are bf16 pairs: X = X_hi + X_lo (fp32 X), W = W_hi + W_lo;
//    Y = X_hi·W_hiᵀ + X_lo·W_hiᵀ + X_hi·W_loᵀ (the lo·lo term is below 2^-16).
//  * tcgen05 fp32 accumulation truncates (mean −2^-25 per accumulation step) → the K loop is cut into
//    segments of ≤ KSEG chunks (≤ 128 accumulation steps, bias ≤ 4e-6); each segment's partial Y is
//    added in fp32 round-to-nearest by the epilogue into its own smem row, and S is formed on the CUDA
//    cores in fp32 per tile, accumulated over ≤ 8 tiles in registers, then flushed to fp64.
#pragma once

namespace ka {
constexpr int BM = 128;            // rows per tile (UMMA M)
constexpr int BK = 64;             // bf16 K elements per chunk
constexpr int KSEG = 16;           // chunks per accumulation segment
constexpr int NCONV = 16;          // converter warps
constexpr int RPW = BM / NCONV;    // rows per converter warp per chunk (8)
constexpr int LPT = RPW / 2;       // float4 loads per converter thread per chunk (4)
constexpr int W_CONV0 = 4;
constexpr int W_CTRL = 4 + NCONV;  // 20: W' TMA ring (lane 0), bf16 X TMA ring (lane 1)
constexpr int W_MMA = W_CTRL + 1;  // 21: MMA issue (own warp: a spinning lane must not delay the producers)
constexpr int NTHREADS = (W_MMA + 1) * 32;
constexpr int SFLUSH = 8;          // tiles between fp32 → fp64 flushes of the S partial
constexpr int PF = 0;              // converter L2-prefetch distance in K chunks (measured: prefetching hurts; off)
constexpr uint32_t XST = BM * 128; // one bf16 X stage (hi or lo)
// XM (X mode): 0 = fp32 X converted by the converter warps, 1 = bf16 X by TMA, 2 = PPCA_F32_SPLIT by TMA
__host__ __device__ constexpr int nst(int MP, int xm) { return xm == 1 ? 4 : (MP <= 64 ? 3 : 2); }
__host__ __device__ constexpr int nws(int MP) { return MP <= 64 ? 4 : 2; }
__host__ __device__ constexpr int ntb(int MP) { return 2 * MP <= 128 ? 4 : 2; }
__host__ __device__ constexpr size_t smem_bytes(int MP, int xm) {
  return 1024 + (size_t)nst(MP, xm) * (xm == 1 ? XST : 2 * XST) + (size_t)nws(MP) * 2 * MP * 128 +
         (size_t)BM * (MP + 4) * 4 + 512;
}
}  // namespace ka

struct KAParams {
  const void* X;          // fp32 or bf16 [n][ld]
  int64_t n, d, ld;
  int m, mp;              // m, m padded to a multiple of 16
  int64_t ntiles, nk;     // row tiles, K chunks
  __nv_bfloat16* YT;      // optional Yᵀ out, bf16 pair [2·mp][ldyt]
  int64_t ldyt;
  double* Spart;          // [gridDim.x][mp][mp] fp64 per-CTA partials (upper triangle used)
  int dbg;                // experiment switches (env PPCA_DBG; 0 in production)
  // K split (kernel A2 only): work item = (tile, K part); with ksplit > 1 the epilogue writes the fp32
  // partial Y of its K part to Ypart [ksplit][n][mp] (no S, no Yᵀ) for a short row window (minibatch step)
  int ksplit = 1;
  int64_t kper = 0;       // K chunks per part
  float* Ypart = nullptr;
  // row-tile list (kernel A2 only): item tiles are tiles[i] instead of i (the row-subsampled refine)
  const int32_t* tiles = nullptr;
};

template <int MP, int XM>
__global__ void __launch_bounds__(ka::NTHREADS, 1)
    xw_tc_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                 const __grid_constant__ CUtensorMap tmXlo, KAParams p) {
  using namespace ka;
  constexpr bool TMAX = XM != 0;                    // X stages filled by TMA (bf16 / split planes)
  constexpr bool LO = XM != 1;                      // an X_lo plane exists (fp32 converted, or split)
  constexpr uint32_t XSTG = LO ? 2 * XST : XST;     // X stage: hi (+ lo)
  constexpr int NST = nst(MP, XM), NWS = nws(MP), NTB = ntb(MP);
  static_assert(smem_bytes(MP, XM) <= 227 * 1024, "kernel A shared memory budget");
  constexpr int NB = 2 * MP;                        // UMMA N: [W_hi; W_lo]
  constexpr uint32_t WST = NB * 128;
  constexpr uint32_t TCOLS = NTB * NB <= 32 ? 32 : (NTB * NB <= 64 ? 64 : (NTB * NB <= 128 ? 128 : (NTB * NB <= 256 ? 256 : 512)));
  constexpr int YS_LD = MP + 4;                     // 16-B aligned rows for LDS.128
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sX = sm;                                 // NST × XSTG
  uint8_t* sW = sX + NST * XSTG;                    // NWS × WST
  float* Ys = reinterpret_cast<float*>(sW + NWS * WST);   // BM × YS_LD (fp32 Y of the current tile)
  uint64_t* bars = reinterpret_cast<uint64_t*>(Ys + BM * YS_LD + 2);
  uint64_t* full = bars;                            // X stage filled (converters / TMA)
  uint64_t* empty = full + NST;                     // X stage consumed (MMA commit)
  uint64_t* wfull = empty + NST;
  uint64_t* wempty = wfull + NWS;
  uint64_t* tfull = wempty + NWS;                   // TMEM segment accumulator ready
  uint64_t* tempty = tfull + NTB;                   // TMEM segment accumulator drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + NTB);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], TMAX ? 1 : NCONV);
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
  if (warp == W_CTRL && lane == 0) {
    tma_prefetch_desc(&tmW);
    if (TMAX) tma_prefetch_desc(&tmX);
    if (XM == 2) tma_prefetch_desc(&tmXlo);
  }
  if (warp == W_MMA) tmem_alloc<TCOLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int64_t t0 = blockIdx.x, tstep = gridDim.x;
  const int64_t nseg = (p.nk + KSEG - 1) / KSEG;    // accumulation segments per tile

  if (warp == W_CTRL || warp == W_MMA) {
    if (warp == W_CTRL && lane == 0) {
      // ---------------------------------------------------------------- W' ring (TMA from L2)
      uint32_t it = 0;
      for (int64_t t = t0; t < p.ntiles && !(p.dbg & 32); t += tstep)
        for (int64_t kc = 0; kc < p.nk; ++kc, ++it) {
          const uint32_t s = it % NWS, ph = (it / NWS) & 1;
          mbar_wait(&wempty[s], ph ^ 1);
          mbar_arrive_expect_tx(&wfull[s], WST);
          tma_load_2d(sW + s * WST, &tmW, &wfull[s], (int32_t)(kc * BK), 0);
        }
    } else if (TMAX && warp == W_CTRL && lane == 1) {
      // ---------------------------------------------------------------- X ring (bf16 X / split planes by TMA)
      const uint64_t pol = policy_evict_first();
      uint32_t it = 0;
      for (int64_t t = t0; t < p.ntiles; t += tstep)
        for (int64_t kc = 0; kc < p.nk; ++kc, ++it) {
          const uint32_t s = it % NST, ph = (it / NST) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          mbar_arrive_expect_tx(&full[s], XSTG);
          tma_load_2d_hint(sX + s * XSTG, &tmX, &full[s], (int32_t)(kc * BK), (int32_t)(t * BM), pol);
          if (XM == 2) tma_load_2d_hint(sX + s * XSTG + XST, &tmXlo, &full[s], (int32_t)(kc * BK), (int32_t)(t * BM), pol);
        }
    } else if (warp == W_MMA && lane == 0) {
      // ---------------------------------------------------------------- MMA issue (one thread)
      constexpr uint32_t ID = idesc(FMT_BF16, FMT_BF16, BM, NB, 0, 0);
      constexpr uint32_t ID_HI = idesc(FMT_BF16, FMT_BF16, BM, MP, 0, 0);
      uint32_t it = 0, sg = 0;
      for (int64_t t = t0; t < p.ntiles; t += tstep)
        for (int64_t g = 0; g < nseg; ++g, ++sg) {
          const uint32_t b = sg % NTB, tph = (sg / NTB) & 1;
          mbar_wait(&tempty[b], tph ^ 1);
          tc_fence_after();
          const uint32_t dcol = tmem + b * NB;
          const int64_t k1 = min(p.nk, (g + 1) * KSEG);
          for (int64_t kc = g * KSEG; kc < k1; ++kc, ++it) {
            const uint32_t s = it % NST, ph = (it / NST) & 1;
            const uint32_t ws = it % NWS, wph = (it / NWS) & 1;
            if (!(p.dbg & 32)) mbar_wait(&wfull[ws], wph);
            mbar_wait(&full[s], ph);
            tc_fence_after();
            if (!(p.dbg & 1)) {
              const uint32_t xa = smem_u32(sX + s * XSTG), wa = smem_u32(sW + ws * WST);
#pragma unroll
              for (int kk = 0; kk < BK / 16; ++kk) {
                // [hi | lo] columns (+)= X_hi·[W_hi; W_lo]ᵀ
                mma_bf16(dcol, smem_desc_sw128(xa + kk * 32, 16, 1024), smem_desc_sw128(wa + kk * 32, 16, 1024), ID,
                         (kc != g * KSEG) || kk != 0);
                // hi columns += X_lo·W_hiᵀ   (fp32 X only)
                if (LO && !(p.dbg & 8))
                  mma_bf16(dcol, smem_desc_sw128(xa + XST + kk * 32, 16, 1024),
                           smem_desc_sw128(wa + kk * 32, 16, 1024), ID_HI, 1);
              }
            }
            mma_commit(&empty[s]);
            mma_commit(&wempty[ws]);
          }
          mma_commit(&tfull[b]);
        }
    }
  } else if (warp >= W_CONV0 && warp < W_CONV0 + NCONV) {
    // ------------------------------------------------------------------ fp32 → bf16 pair converters
    if (XM == 0) {
      const float* X = reinterpret_cast<const float*>(p.X);
      const int cw = warp - W_CONV0;
      const int sub = lane >> 4, cl = lane & 15;
      // chunk ci of this CTA = (tile t0 + ⌊ci/nk⌋·tstep, K chunk ci mod nk), the MMA order; load and
      // store cursors advance incrementally; three register buffers keep two chunks of loads in flight.
      const int64_t nchunks = ((p.ntiles - t0 + tstep - 1) / tstep) * p.nk;
      int64_t lt = t0, lk = 0;
      uint32_t ss = 0, sph = 0;
      // L2 prefetch cursor, PF chunks ahead of the loads (one prefetch per 128-B line: lanes cl % 8 == 0)
      int64_t pt = t0, pk = 0, pci = 0;
      auto prefetch_next = [&]() {
        if (pci >= nchunks) return;
        const int64_t row0 = pt * BM + cw * RPW + sub;
        const int64_t col = pk * BK + cl * 4;
        if ((cl & 7) == 0 && col < p.d) {
#pragma unroll
          for (int i = 0; i < LPT; ++i)
            if (row0 + 2 * i < p.n) prefetch_l2(X + (row0 + 2 * i) * p.ld + col);
        }
        if (++pk == p.nk) { pk = 0; pt += tstep; }
        ++pci;
      };
      for (int i = 0; i < PF; ++i) prefetch_next();
      auto load = [&](int64_t ci, float4 (&r)[LPT]) {
        if (ci >= nchunks) return;
        if (PF) prefetch_next();
        const int64_t row0 = lt * BM + cw * RPW + sub;
        const int64_t col = lk * BK + cl * 4;
        const float* base = X + row0 * p.ld + col;
        const bool colok = col < p.d;
#pragma unroll
        for (int i = 0; i < LPT; ++i) {
          float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
          if (colok && row0 + 2 * i < p.n) v = __ldcs(reinterpret_cast<const float4*>(base + 2 * i * p.ld));
          r[i] = v;
        }
        if (++lk == p.nk) { lk = 0; lt += tstep; }
      };
      auto store = [&](const float4 (&r)[LPT]) {
        const uint32_t s = ss, ph = sph;
        if (++ss == NST) { ss = 0; sph ^= 1; }
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* st = sX + s * XSTG;
        if (!(p.dbg & 4)) {
#pragma unroll
          for (int i = 0; i < LPT; ++i) {
            const uint32_t off = sw128(cw * RPW + 2 * i + sub, cl * 8);
            const uint2 hi = pack4_bf16(r[i]);
            *reinterpret_cast<uint2*>(st + off) = hi;
            if (!(p.dbg & 16)) *reinterpret_cast<uint2*>(st + XST + off) = pack4_bf16(residual_bf16(r[i], hi));
          }
        } else {
          float acc = 0.f;   // keep the loads live without touching shared memory
#pragma unroll
          for (int i = 0; i < LPT; ++i) acc += r[i].x + r[i].y + r[i].z + r[i].w;
          if (acc == 1234.5f) *reinterpret_cast<float*>(st) = acc;
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[s]);
      };
      float4 A[LPT], B[LPT], Cb[LPT];
      load(0, A);
      load(1, B);
      for (int64_t ci = 0; ci < nchunks; ci += 3) {
        load(ci + 2, Cb);
        store(A);
        if (ci + 1 >= nchunks) break;
        load(ci + 3, A);
        store(B);
        if (ci + 2 >= nchunks) break;
        load(ci + 4, B);
        store(Cb);
      }
    }
  } else if (warp < 4) {
    // ------------------------------------------------------------------ epilogue (128 threads = 128 rows)
    const int tid = threadIdx.x;
    // S: thread t owns 4×4 blocks (bi ≤ bj) b = t, t+128, … of the upper triangle
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
    // fp32 block sums live in registers for ≤ SFLUSH tiles when they fit (m ≤ 64); for larger m every
    // tile's block sums go straight to the fp64 slot (m > 64 means d is large and a tile costs far more).
    constexpr bool SREG = MAXB <= 2;
    constexpr int SFL = SREG ? SFLUSH : 1;
    float sacc[SREG ? MAXB : 1][16];
#pragma unroll
    for (int q = 0; q < MAXB; ++q)
#pragma unroll
      for (int e = 0; e < 16; ++e) sacc[q][e] = 0.f;
    double* Sp = p.Spart + (int64_t)blockIdx.x * MP * MP;
#pragma unroll
    for (int q = 0; q < MAXB; ++q)
      if (bi_[q] >= 0)
        for (int e = 0; e < 16; ++e) Sp[(4 * bi_[q] + e / 4) * MP + 4 * bj_[q] + e % 4] = 0.0;
    auto flush = [&]() {
#pragma unroll
      for (int q = 0; q < MAXB; ++q)
        if (bi_[q] >= 0)
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            Sp[(4 * bi_[q] + e / 4) * MP + 4 * bj_[q] + e % 4] += (double)sacc[q][e];
            sacc[q][e] = 0.f;
          }
    };
    float* yrow = Ys + tid * YS_LD;
    uint32_t sg = 0, tcount = 0;
    for (int64_t t = t0; t < p.ntiles; t += tstep) {
      for (int64_t g = 0; g < nseg; ++g, ++sg) {
        const uint32_t b = sg % NTB, tph = (sg / NTB) & 1;
        mbar_wait(&tfull[b], tph);
        tc_fence_after();
#pragma unroll 1
        for (int c0 = 0; c0 < MP; c0 += 8) {
          float v[8], w[8];
          const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + b * NB + c0;
          tmem_ld8(ta, v);          // X'·W_hiᵀ
          tmem_ld8(ta + MP, w);     // X'·W_loᵀ
#pragma unroll
          for (int j = 0; j < 8; j += 4) {
            float4 cur = g == 0 ? make_float4(0.f, 0.f, 0.f, 0.f) : *reinterpret_cast<const float4*>(yrow + c0 + j);
            cur.x += v[j] + w[j];
            cur.y += v[j + 1] + w[j + 1];
            cur.z += v[j + 2] + w[j + 2];
            cur.w += v[j + 3] + w[j + 3];
            *reinterpret_cast<float4*>(yrow + c0 + j) = cur;
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[b]);
      }
      // the tile's Y row is complete in yrow (fp32, round-to-nearest sums of the segments)
      const int64_t grow = t * BM + tid;
      if (p.YT && grow < p.ldyt) {           // Yᵀ as a bf16 pair [Y_hi; Y_lo] (rows ≥ n are zero)
#pragma unroll 4
        for (int j = 0; j < MP; ++j) {
          const float y = yrow[j];
          const __nv_bfloat16 hi = __float2bfloat16_rn(y);
          p.YT[(int64_t)j * p.ldyt + grow] = hi;
          p.YT[(int64_t)(MP + j) * p.ldyt + grow] = __float2bfloat16_rn(y - __bfloat162float(hi));
        }
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (!(p.dbg & 2)) {
#pragma unroll
        for (int q = 0; q < MAXB; ++q) {
          if (bi_[q] < 0) continue;
          const float* ya = Ys + 4 * bi_[q];
          const float* yb = Ys + 4 * bj_[q];
          float s16[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) s16[e] = 0.f;
#pragma unroll 4
          for (int r = 0; r < BM; ++r) {
            const float4 a = *reinterpret_cast<const float4*>(ya + r * YS_LD);
            const float4 c = *reinterpret_cast<const float4*>(yb + r * YS_LD);
            const float av[4] = {a.x, a.y, a.z, a.w}, cv[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
            for (int x = 0; x < 4; ++x)
#pragma unroll
              for (int y = 0; y < 4; ++y) s16[x * 4 + y] = fmaf(av[x], cv[y], s16[x * 4 + y]);
          }
          if (SREG) {
#pragma unroll
            for (int e = 0; e < 16; ++e) sacc[q][e] += s16[e];
          } else {
#pragma unroll
            for (int e = 0; e < 16; ++e) Sp[(4 * bi_[q] + e / 4) * MP + 4 * bj_[q] + e % 4] += (double)s16[e];
          }
        }
      }
      if (SREG && ++tcount == SFL) {
        tcount = 0;
        flush();
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
    }
    if (SREG) flush();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == W_MMA) tmem_dealloc<TCOLS>(tmem);
}
