// tc_xw2.cuh — kernel A for TMA-staged X (a bf16 X, or the two bf16 planes of a PPCA_F32_SPLIT X):
//   Y_t = X_t·W'ᵀ  and  S += Y_tᵀY_t   (§8 rows a2 / a7; PAPER.md L61-63 product, L260-269 projected Gram).
//
// Persistent, one CTA per SM, 7 warps: 0-3 epilogue (TMEM lane quadrants, thread = tile row), 4 W' TMA
// ring, 5 X TMA ring, 6 MMA issue (owns TMEM).  No CUDA-core
// conversion: TMA writes the bf16 planes straight into SWIZZLE_128B atoms that the UMMA descriptors read.
//
// Product 1 per 128-row tile and 64-column K chunk (UMMA M=128, K=16):  [hi | lo] columns (+)= X_hi·[W_hi; W_lo]ᵀ
// (N = 2·MP) and, for a split X, hi columns += X_lo·W_hiᵀ.  The K loop is cut into segments of ≤ KSEG
// chunks (tcgen05's fp32 accumulate truncates; tests/tc_accum_test.cu) whose partial Y the epilogue adds
// in fp32 round-to-nearest.
//
// S for MP = 64 runs on the tensor cores: the epilogue writes Y_t as bf16 [Y_hi | Y_lo] rows into an
// MN-major SW128 tile and one UMMA chain (M = N = 128, K = 128 rows) forms D = [Y_hi|Y_lo]ᵀ[Y_hi|Y_lo];
// thread i drains row i of D as R_i = D[i][0:64] + D[i][64:128], so rows i and i+64 together hold
// (Y_hi + Y_lo)ᵀ(Y_hi + Y_lo).  Partials: fp32 registers over ≤ SFLUSH tiles, then fp64 per CTA
// (Spart [cta][2·MP][MP]); reduce_spart2 sums them in a fixed order.  Other MP keep the CUDA-core S of
// kernel A (4×4 register blocks over the fp32 Y rows).
#pragma once

namespace ka2 {
constexpr int BM = 128;            // rows per tile (UMMA M)
constexpr int BK = 64;             // bf16 K elements per chunk (one 128-byte swizzle row)
constexpr int KSEG = 16;           // chunks per accumulation segment
constexpr int SFLUSH = 8;          // tiles between fp32 → fp64 flushes of the S partial
// warps 0-3 epilogue, 4 W' producer, 5 X producer, 6 MMA issuer (separate warps: a lane spinning on an
// mbarrier must not delay the other roles' lanes of the same warp)
constexpr int W_WPROD = 4, W_XPROD = 5, W_MMA = 6;
constexpr int NTHREADS = 7 * 32;
constexpr uint32_t XST = BM * 128; // one bf16 plane stage (128 rows × 64 columns)
constexpr uint32_t YBLK = BM * 128;   // one 64-feature block of the Y operand tile
constexpr int XPF = 0;             // X chunks prefetched into L2 ahead of the TMA loads (measured: hurts)

template <int MP, int XM, bool PAIR = false>
struct Cfg {
  static constexpr bool SMMA = MP == 64;                        // S on the tensor cores
  static constexpr int NB = 2 * MP;                             // product-1 UMMA N: [W_hi; W_lo]
  static constexpr int NTB = SMMA ? 2 : (NB <= 128 ? 4 : 2);    // TMEM Y segment buffers
  static constexpr int SCOL0 = NTB * NB;                        // TMEM column of the S accumulator
  static constexpr int TUSED = NTB * NB + (SMMA ? 128 : 0);
  static constexpr uint32_t TCOLS =
      TUSED <= 32 ? 32 : (TUSED <= 64 ? 64 : (TUSED <= 128 ? 128 : (TUSED <= 256 ? 256 : 512)));
  static constexpr int PLANES = XM == 2 ? 2 : 1;
  static constexpr uint32_t XSTG = PLANES * XST;
  // W' stages: a 2·MP-row W' chunk is as large as (MP = 64) or twice (MP = 128) the X chunk it multiplies and
  // comes from L2, so its ring must cover L2 latency too (measured on C5: 2 stages starve the MMA)
  // PAIR (2-CTA UMMA, M = 256): each CTA of the pair holds half of every W' chunk (NB/2 rows)
  // small m: the W' chunk is only 2·MP rows (4 KB at MP = 16) and, at huge d (W' beyond L2), comes from HBM, so
  // the ring keeps ≥ 64 KB in flight (up to 16 stages) instead of 4 stages
  static constexpr uint32_t WST = (PAIR ? NB / 2 : NB) * 128;
  static constexpr int NWS = PAIR ? 4 : (MP < 64 ? (int)(65536 / WST > 16 ? 16 : 65536 / WST) : (MP == 64 ? 4 : (XM == 1 ? 3 : 2)));
  // fp32 Y rows for the CUDA-core S (the tensor-core S keeps the segment sums in registers)
  static constexpr size_t YS = SMMA ? 0 : (size_t)BM * (MP + 4) * 4;
  static constexpr size_t YSM = SMMA ? (size_t)2 * YBLK : 0;    // bf16 [Y_hi | Y_lo] operand tile
  static constexpr size_t FIXED = 1024 + (size_t)NWS * WST + YSM + YS + 512;
  static constexpr int NST_FIT = (int)((227 * 1024 - FIXED) / XSTG);
  static constexpr int NST = NST_FIT > 6 ? 6 : NST_FIT;
  static constexpr size_t SMEM = FIXED + (size_t)NST * XSTG;
  static constexpr int SPROWS = SMMA ? 2 * MP : MP;             // rows of a CTA's S partial
};
}  // namespace ka2

// PAIR: CTA pairs (cluster of 2) share one 2-CTA UMMA (M = 256 rows: tile 2q+r in CTA r; W' split by N across
// the pair, so each CTA streams half of every W' chunk from L2).  Rank 1's TMA loads complete on rank 0's
// stage barriers (.cta_group::2), rank 0 issues the MMAs, completions are multicast to both CTAs' barriers;
// each CTA drains its own TMEM rows (rank 1's epilogue releases rank 0's TMEM-empty barrier remotely).  Used for MP = 128 with bf16 X (C5), whole tiles, no tile list.
template <int MP, int XM, bool PAIR = false>
__global__ void __launch_bounds__(ka2::NTHREADS, 1)
    xw_tma_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                  const __grid_constant__ CUtensorMap tmXlo, KAParams p) {
  pdl_wait();   // a programmatic dependent launch: inputs of the previous grid visible
  using namespace ka2;
  using CF = Cfg<MP, XM, PAIR>;
  static_assert(!PAIR || (MP == 128 && XM == 1), "kernel A2 pairs: MP = 128, bf16 X");
  constexpr int NST = CF::NST, NWS = CF::NWS, NTB = CF::NTB, NB = CF::NB;
  constexpr uint32_t XSTG = CF::XSTG, WST = CF::WST, TCOLS = CF::TCOLS;
  constexpr bool SMMA = CF::SMMA, LO = XM == 2;
  constexpr int YS_LD = MP + 4;
  static_assert(CF::NST >= 2, "kernel A (TMA): at least two X stages");
  static_assert(CF::SMEM <= 227 * 1024, "kernel A (TMA) shared memory budget");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sX = sm;                                  // NST × XSTG
  uint8_t* sW = sX + NST * XSTG;                     // NWS × WST
  uint8_t* sY = sW + NWS * WST;                      // YSM: [Y_hi block | Y_lo block]
  float* Ys = reinterpret_cast<float*>(sY + CF::YSM);   // BM × YS_LD
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(Ys) + CF::YS);
  uint64_t* full = bars;
  uint64_t* empty = full + NST;
  uint64_t* wfull = empty + NST;
  uint64_t* wempty = wfull + NWS;
  uint64_t* tfull = wempty + NWS;
  uint64_t* tempty = tfull + NTB;
  uint64_t* yfull = tempty + NTB;                    // Y operand tile written (4 epilogue warps)
  uint64_t* sfull = yfull + 1;                       // S chain of a tile complete (MMA commit)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sfull + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < NWS; ++s) {
      mbar_init(&wfull[s], 1);
      mbar_init(&wempty[s], 1);
    }
    for (int b = 0; b < NTB; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], PAIR ? 8 : 4);
    }
    mbar_init(yfull, 4);
    mbar_init(sfull, 1);
    fence_barrier_init();
  }
  if (warp == W_XPROD && lane == 0) {
    tma_prefetch_desc(&tmW);
    tma_prefetch_desc(&tmX);
    if (LO) tma_prefetch_desc(&tmXlo);
  }
  if (warp == W_MMA) {
    if constexpr (PAIR) tmem_alloc_pair<TCOLS>(tmem_slot);
    else tmem_alloc<TCOLS>(tmem_slot);
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) cluster_barrier();            // the peer's barriers exist before any remote arrive
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t rank = PAIR ? pair_rank() : 0;
  // work item = (row tile, K part): t = it / ksplit, chunks [k0, k1) (ksplit = 1: whole tiles); PAIR: item =
  // tile pair q, this CTA's tile 2q + rank
  const int64_t nitems = PAIR ? (p.ntiles + 1) / 2 : p.ntiles * p.ksplit;
  const int64_t i0 = PAIR ? blockIdx.x / 2 : blockIdx.x, istep = PAIR ? gridDim.x / 2 : gridDim.x;
  const bool partial = p.ksplit > 1;
  auto item = [&](int64_t it, int64_t& t, int64_t& k0, int64_t& k1, int64_t& nseg) {
    if constexpr (PAIR) {
      t = 2 * it + rank;
      k0 = 0;
      k1 = p.nk;
      nseg = (k1 - k0 + KSEG - 1) / KSEG;
      return;
    }
    t = p.tiles ? (int64_t)p.tiles[it / p.ksplit] : it / p.ksplit;
    k0 = (it % p.ksplit) * p.kper;
    k1 = min(p.nk, k0 + p.kper);
    nseg = k1 > k0 ? (k1 - k0 + KSEG - 1) / KSEG : 0;
  };

  if (warp >= W_WPROD) {
    if (warp == W_WPROD && lane == 0) {
      // ---------------------------------------------------------------- W' ring (TMA, L2-resident)
      uint32_t it = 0;
      for (int64_t wi = i0; wi < nitems && !(p.dbg & 32); wi += istep) {
        int64_t t, k0, k1, ns;
        item(wi, t, k0, k1, ns);
        for (int64_t kc = k0; kc < k1; ++kc, ++it) {
          const uint32_t s = it % NWS, ph = (it / NWS) & 1;
          mbar_wait(&wempty[s], ph ^ 1);
          if (PAIR && rank == 1) {                    // rank 1's half signals rank 0's barrier
            tma_load_2d_to_peer_bar(sW + s * WST, &tmW, &wfull[s], 0, (int32_t)(kc * BK), (int32_t)(NB / 2),
                                    policy_evict_last());
          } else {
            mbar_arrive_expect_tx(&wfull[s], PAIR ? 2 * WST : WST);
            tma_load_2d(sW + s * WST, &tmW, &wfull[s], (int32_t)(kc * BK), 0);
          }
        }
      }
    } else if (warp == W_XPROD && lane == 0) {
      // ---------------------------------------------------------------- X ring (hi [+ lo] planes)
      const uint64_t pol = policy_evict_first();
      uint32_t it = 0;
      for (int64_t xi = i0; xi < nitems; xi += istep) {
        int64_t t, k0, k1, ns;
        item(xi, t, k0, k1, ns);
        for (int64_t kc = k0; kc < k1; ++kc, ++it) {
          const uint32_t s = it % NST, ph = (it / NST) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          if (PAIR && rank == 1) {
            tma_load_2d_to_peer_bar(sX + s * XSTG, &tmX, &full[s], 0, (int32_t)(kc * BK), (int32_t)(t * BM), pol);
            continue;
          }
          mbar_arrive_expect_tx(&full[s], PAIR ? 2 * XSTG : ((p.dbg & 64) ? XST : XSTG));
          tma_load_2d_hint(sX + s * XSTG, &tmX, &full[s], (int32_t)(kc * BK), (int32_t)(t * BM), pol);
          if (LO && !(p.dbg & 64))
            tma_load_2d_hint(sX + s * XSTG + XST, &tmXlo, &full[s], (int32_t)(kc * BK), (int32_t)(t * BM), pol);
        }
      }
    } else if (PAIR && warp == W_MMA && rank == 1) {
      // pair rank 1 issues no MMAs: its stages signal rank 0's barriers directly (TMA .cta_group::2)
    } else if (warp == W_MMA && lane == 0) {
      // ---------------------------------------------------------------- MMA issue (one thread)
      constexpr uint32_t ID = idesc(FMT_BF16, FMT_BF16, PAIR ? 2 * BM : BM, NB, 0, 0);
      constexpr uint32_t ID_HI = idesc(FMT_BF16, FMT_BF16, BM, MP, 0, 0);
      constexpr uint32_t ID_S = idesc(FMT_BF16, FMT_BF16, 128, 128, 1, 1);   // Y tile MN-major
      auto issue_s = [&](uint32_t j) {
        mbar_wait(yfull, j & 1);
        tc_fence_after();
        const uint32_t ya = smem_u32(sY);
#pragma unroll
        for (int kk = 0; kk < BM / 16; ++kk) {
          const uint64_t dy = smem_desc_sw128(ya + kk * 2048, YBLK, 1024);
          if (!(p.dbg & 2)) mma_bf16(tmem + CF::SCOL0, dy, dy, ID_S, kk != 0);
        }
        mma_commit(sfull);
      };
      uint32_t it = 0, sg = 0, lt = 0;
      for (int64_t mi = i0; mi < nitems; mi += istep, ++lt) {
        int64_t t, k0, k1, nseg;
        item(mi, t, k0, k1, nseg);
        for (int64_t g = 0; g < nseg; ++g, ++sg) {
          const uint32_t b = sg % NTB, tph = (sg / NTB) & 1;
          if constexpr (PAIR) mbar_wait_cluster(&tempty[b], tph ^ 1);
          else mbar_wait(&tempty[b], tph ^ 1);
          tc_fence_after();
          const uint32_t dcol = tmem + b * NB;
          const int64_t g0 = k0 + g * KSEG, g1 = min(k1, g0 + KSEG);
          for (int64_t kc = g0; kc < g1; ++kc, ++it) {
            const uint32_t s = it % NST, ph = (it / NST) & 1;
            const uint32_t ws = it % NWS, wph = (it / NWS) & 1;
            if (!(p.dbg & 32)) mbar_wait(&wfull[ws], wph);
            mbar_wait(&full[s], ph);
            tc_fence_after();
            const uint32_t xa = smem_u32(sX + s * XSTG), wa = smem_u32(sW + ws * WST);
#pragma unroll
            for (int kk = 0; kk < BK / 16 && !(p.dbg & 1); ++kk) {
              if constexpr (PAIR) {
                mma_bf16_pair(dcol, smem_desc_sw128(xa + kk * 32, 16, 1024), smem_desc_sw128(wa + kk * 32, 16, 1024),
                              ID, (kc != g0) || kk != 0);
              } else {
                mma_bf16(dcol, smem_desc_sw128(xa + kk * 32, 16, 1024), smem_desc_sw128(wa + kk * 32, 16, 1024), ID,
                         (kc != g0) || kk != 0);
                if (LO)
                  mma_bf16(dcol, smem_desc_sw128(xa + XST + kk * 32, 16, 1024),
                           smem_desc_sw128(wa + kk * 32, 16, 1024), ID_HI, 1);
              }
            }
            if constexpr (PAIR) {
              mma_commit_pair(&empty[s], 3);
              mma_commit_pair(&wempty[ws], 3);
            } else {
              mma_commit(&empty[s]);
              mma_commit(&wempty[ws]);
            }
          }
          if constexpr (PAIR) mma_commit_pair(&tfull[b], 3);
          else mma_commit(&tfull[b]);
        }
        // S of the previous tile, issued behind this tile's product 1 so the tensor pipe never waits
        // for the epilogue
        if (SMMA && !partial && lt > 0) issue_s(lt - 1);
      }
      if (SMMA && !partial && lt > 0) issue_s(lt - 1);
    }
  } else {
    // ------------------------------------------------------------------ epilogue (128 threads = 128 rows)
    const int tid = threadIdx.x;
    double* Sp = p.Spart + (int64_t)blockIdx.x * CF::SPROWS * MP;
    for (int e = tid; e < CF::SPROWS * MP; e += 128) Sp[e] = 0.0;
    asm volatile("bar.sync 1, 128;" ::: "memory");
    float* yrow = Ys + tid * YS_LD;
    const uint32_t tl = (uint32_t)(warp * 32) << 16;   // this warp's TMEM lane quadrant
    uint32_t sg = 0, lt = 0;

    if constexpr (SMMA) {
      float sacc[MP];
#pragma unroll
      for (int j = 0; j < MP; ++j) sacc[j] = 0.f;
      int pending = 0;                                   // drained tiles not yet flushed to fp64
      auto flush = [&]() {
        double* row = Sp + tid * MP;
#pragma unroll
        for (int j = 0; j < MP; ++j) {
          row[j] += (double)sacc[j];
          sacc[j] = 0.f;
        }
        pending = 0;
      };
      auto drain = [&](uint32_t j) {                     // R_tid = D[tid][0:64] + D[tid][64:128]
        mbar_wait(sfull, j & 1);
        tc_fence_after();
#pragma unroll
        for (int c0 = 0; c0 < MP; c0 += 16) {
          float a[16], b2[16];
          tmem_ld16(tmem + tl + CF::SCOL0 + c0, a);
          tmem_ld16(tmem + tl + CF::SCOL0 + MP + c0, b2);
#pragma unroll
          for (int q = 0; q < 16; ++q) sacc[c0 + q] += a[q] + b2[q];
        }
        if (++pending == SFLUSH) flush();
      };
      for (int64_t ei = i0; ei < nitems; ei += istep) {
        int64_t t, k0, k1, nseg;
        item(ei, t, k0, k1, nseg);
        float y[MP];
#pragma unroll
        for (int j = 0; j < MP; ++j) y[j] = 0.f;
        for (int64_t g = 0; g < nseg; ++g, ++sg) {
          const uint32_t b = sg % NTB, tph = (sg / NTB) & 1;
          mbar_wait(&tfull[b], tph);
          tc_fence_after();
#pragma unroll
          for (int c0 = 0; c0 < MP; c0 += 8) {
            float v[8], w[8];
            tmem_ld8(tmem + tl + b * NB + c0, v);        // X'·W_hiᵀ
            tmem_ld8(tmem + tl + b * NB + MP + c0, w);   // X'·W_loᵀ
#pragma unroll
            for (int j = 0; j < 8; ++j) y[c0 + j] = y[c0 + j] + (v[j] + w[j]);
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (PAIR && rank == 1) mbar_arrive_peer(&tempty[b], 0);
            else mbar_arrive(&tempty[b]);
          }
        }
        const int64_t grow = t * BM + tid;
        if (partial) {                                   // K part of a row window: fp32 partial Y out
          if (grow < p.n) {
            float4* dst = reinterpret_cast<float4*>(p.Ypart + ((ei % p.ksplit) * p.n + grow) * MP);
#pragma unroll
            for (int j = 0; j < MP; j += 4) dst[j / 4] = make_float4(y[j], y[j + 1], y[j + 2], y[j + 3]);
          }
          continue;
        }
        if (p.YT && grow < p.ldyt) {                     // Yᵀ as a bf16 pair [Y_hi; Y_lo] (rows ≥ n are zero)
#pragma unroll
          for (int j = 0; j < MP; ++j) {
            const __nv_bfloat16 hi = __float2bfloat16_rn(y[j]);
            p.YT[(int64_t)j * p.ldyt + grow] = hi;
            p.YT[(int64_t)(MP + j) * p.ldyt + grow] = __float2bfloat16_rn(y[j] - __bfloat162float(hi));
          }
        }
        if (lt > 0) drain(lt - 1);                       // S(t-1) is read before the Y tile is rewritten
        // Y tile row `tid`: [Y_hi (64 features) | Y_lo (64 features)], MN-major SW128 (16-B chunks)
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) {
          uint32_t h[4], l[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float a0 = y[ch * 8 + 2 * q], a1 = y[ch * 8 + 2 * q + 1];
            const __nv_bfloat162 hv = __floats2bfloat162_rn(a0, a1);
            const __nv_bfloat162 lv =
                __floats2bfloat162_rn(a0 - __low2float(hv), a1 - __high2float(hv));
            h[q] = *reinterpret_cast<const uint32_t*>(&hv);
            l[q] = *reinterpret_cast<const uint32_t*>(&lv);
          }
          const uint32_t off = (uint32_t)(tid >> 3) * 1024u + (uint32_t)(tid & 7) * 128u + ((ch ^ (tid & 7)) << 4);
          *reinterpret_cast<uint4*>(sY + off) = make_uint4(h[0], h[1], h[2], h[3]);
          *reinterpret_cast<uint4*>(sY + YBLK + off) = make_uint4(l[0], l[1], l[2], l[3]);
        }
        fence_proxy_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(yfull);
        ++lt;
      }
      if (lt > 0) drain(lt - 1);
      if (pending) flush();
    } else {
      // CUDA-core S: thread t owns 4×4 blocks (bi ≤ bj) b = t, t+128, … of the upper triangle
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
      for (int64_t ei = i0; ei < nitems; ei += istep, ++lt) {
        int64_t t, k0, k1, nseg;
        item(ei, t, k0, k1, nseg);
        if (nseg == 0)
          for (int j = 0; j < MP; ++j) yrow[j] = 0.f;
        for (int64_t g = 0; g < nseg; ++g, ++sg) {
          const uint32_t b = sg % NTB, tph = (sg / NTB) & 1;
          mbar_wait(&tfull[b], tph);
          tc_fence_after();
#pragma unroll 1
          for (int c0 = 0; c0 < MP; c0 += 8) {
            float v[8], w[8];
            tmem_ld8(tmem + tl + b * NB + c0, v);
            tmem_ld8(tmem + tl + b * NB + MP + c0, w);
#pragma unroll
            for (int j = 0; j < 8; ++j) yrow[c0 + j] = (g == 0 ? 0.f : yrow[c0 + j]) + (v[j] + w[j]);
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (PAIR && rank == 1) mbar_arrive_peer(&tempty[b], 0);
            else mbar_arrive(&tempty[b]);
          }
        }
        const int64_t grow = t * BM + tid;
        if (partial) {
          if (grow < p.n) {
            float4* dst = reinterpret_cast<float4*>(p.Ypart + ((ei % p.ksplit) * p.n + grow) * MP);
            for (int j = 0; j < MP; j += 4) dst[j / 4] = *reinterpret_cast<const float4*>(yrow + j);
          }
          continue;
        }
        if (p.YT && grow < p.ldyt) {
#pragma unroll 4
          for (int j = 0; j < MP; ++j) {
            const float yv = yrow[j];
            const __nv_bfloat16 hi = __float2bfloat16_rn(yv);
            p.YT[(int64_t)j * p.ldyt + grow] = hi;
            p.YT[(int64_t)(MP + j) * p.ldyt + grow] = __float2bfloat16_rn(yv - __bfloat162float(hi));
          }
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
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
              for (int z = 0; z < 4; ++z) s16[x * 4 + z] = fmaf(av[x], cv[z], s16[x * 4 + z]);
          }
#pragma unroll
          for (int e = 0; e < 16; ++e) Sp[(4 * bi_[q] + e / 4) * MP + 4 * bj_[q] + e % 4] += (double)s16[e];
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) {
    cluster_barrier();                                // no remote arrive may target an exited CTA
    if (warp == W_MMA) tmem_dealloc_pair<TCOLS>(tmem);
  } else {
    if (warp == W_MMA) tmem_dealloc<TCOLS>(tmem);
  }
}
