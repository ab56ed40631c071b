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
// four consecutive elements per thread (d % 8 == 0 on the tensor-core path): 16-byte loads / stores
__global__ void prep_w_kernel(const float* __restrict__ W, int m, int mp, int64_t d, __nv_bfloat16* __restrict__ Wb,
                              float* __restrict__ Wr) {
  pdl_enter();
  const int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (e >= (int64_t)mp * d) return;
  const int64_t i = e / d;
  const float4 v = i < m ? __ldg(reinterpret_cast<const float4*>(W + e)) : make_float4(0.f, 0.f, 0.f, 0.f);
  const uint2 hi = pack4_bf16(v);
  const uint2 lo = pack4_bf16(residual_bf16(v, hi));
  *reinterpret_cast<uint2*>(Wb + e) = hi;
  *reinterpret_cast<uint2*>(Wb + e + (int64_t)mp * d) = lo;
  if (i < m) {
    *reinterpret_cast<float4*>(Wr + e) =
        make_float4(__uint_as_float(hi.x << 16) + __uint_as_float(lo.x << 16),
                    __uint_as_float(hi.x & 0xffff0000u) + __uint_as_float(lo.x & 0xffff0000u),
                    __uint_as_float(hi.y << 16) + __uint_as_float(lo.y << 16),
                    __uint_as_float(hi.y & 0xffff0000u) + __uint_as_float(lo.y & 0xffff0000u));
  }
}

// ============================================================================ kernel A (tc_xw.cuh)
#include "tc_xw.cuh"

// S[i][j] = S[j][i] = Σ_cta Spart[cta][pair(i,j)]  (fixed order, fp64)
// Block = 32 outputs (lanes) × 8 warps; warp w sums partials c ≡ w (mod 8), then the 8 warp sums are
// added in warp order — a fixed order, so the result is deterministic.
__global__ void __launch_bounds__(256) reduce_spart_kernel(const double* __restrict__ Spart, int nparts, int mp, int m,
                                                           double* __restrict__ S) {
  pdl_enter();
  __shared__ double part[8][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int e = blockIdx.x * 32 + lane;
  double s = 0.0;
  if (e < m * m) {
    const int i = e / m, j = e % m;
    const int idx = min(i, j) * mp + max(i, j);   // partials hold the upper triangle, dense [mp][mp]
    s = sum_in_order<8>(warp, nparts, 8, [&](int64_t c) { return Spart[c * mp * mp + idx]; });
  }
  part[warp][lane] = s;
  __syncthreads();
  if (warp == 0 && e < m * m) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += part[w][lane];
    S[e] = t;
  }
}

// ============================================================================ kernel A, TMA-staged X (tc_xw2.cuh)
#include "tc_xw2.cuh"

// S[i][j] = S[j][i] = Σ_cta (Sp[cta][a][b] + Sp[cta][a + mp][b]),  a = min(i,j), b = max(i,j)
// (S partials of the tensor-core S: rows a and a+mp hold the hi- and lo-row halves of D; fixed order)
__global__ void __launch_bounds__(256) reduce_spart2_kernel(const double* __restrict__ Spart, int nparts, int mp,
                                                            int m, double* __restrict__ S) {
  pdl_enter();
  __shared__ double part[8][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int e = blockIdx.x * 32 + lane;
  double s = 0.0;
  if (e < m * m) {
    const int i = e / m, j = e % m;
    const int a = min(i, j), b = max(i, j);
    s = sum_in_order<8>(warp, nparts, 8, [&](int64_t c) {
      const double* P = Spart + c * 2 * mp * mp;
      return P[a * mp + b] + P[(a + mp) * mp + b];
    });
  }
  part[warp][lane] = s;
  __syncthreads();
  if (warp == 0 && e < m * m) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += part[w][lane];
    S[e] = t;
  }
}

// ============================================================================ fused power pass (tc_fused.cuh)
#include "tc_fused.cuh"
#include "tc_pair.cuh"

// ============================================================================ kernel B (tc_xty.cuh)
#include "tc_xty.cuh"

// Z[j][x] = Σ_g Zp[g][x][j], g in order (fixed, deterministic): two kernels, for many row groups (the fused
// power passes, nrg ≈ 36-74: 8 warps split the partials of a column) and for few (the minibatch windows).
// Z[j][x] = Σ_g Zp[g][x][j]: block (x, 32 consecutive j), warp w sums g ≡ w (mod 8) (8 loads in flight),
// the 8 warp sums are added in warp order.
// Z's layout: plain [m][d] (ds = d) or d-blocked [d/ds][m][ds] (the slices of the distributed CholQR, §6):
// element (j, x) lives at ((x / ds)·m + j)·ds + x % ds
__device__ __forceinline__ int64_t z_index(int j, int64_t x, int m, int64_t ds) {
  return ((x / ds) * m + j) * ds + x % ds;
}

__global__ void __launch_bounds__(256) reduce_zp_cols_kernel(const float* __restrict__ Zp, int64_t nrg, int64_t dpad,
                                                             int mp, int m, int64_t d, float* __restrict__ Z, int64_t ds) {
  pdl_enter();
  __shared__ double part[8][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t x = blockIdx.x;
  const int j = blockIdx.y * 32 + lane;
  double s = 0.0;
  if (j < m)
    s = sum_in_order<8>(warp, nrg, 8, [&](int64_t g) { return (double)Zp[(g * dpad + x) * mp + j]; });
  part[warp][lane] = s;
  __syncthreads();
  if (warp == 0 && j < m) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += part[w][lane];
    Z[z_index(j, x, m, ds)] = (float)t;
  }
}

// Z[j][x] = Σ_g Zp[g][x][j] for a few row groups (the short windows of the minibatch steps and C5's kernel B,
// nrg ≤ 16): thread = 4 consecutive features of CPT columns (one float4 per partial and column, 16 loads in
// flight: CPT = 4 for nrg ≤ 4), sums in g order in fp64; a block covers CPT·256·4/mp ≤ 64 columns and leaves
// through shared memory as runs of Z's rows (C5, nrg = 4, mp = 128: 32-column blocks write whole 128-byte lines
// of every feature row instead of 32-byte sectors; same sums, same bits).
// The partial loads go through cp.async into a per-thread staging slot ([slot][thread] float4: conflict-free), one
// wait for all 16: in flight together by construction.  Register loads did not stay that way — with the loads under
// the predicate of their use, and also with unconditional loads, ptxas places every conversion right behind its load
// to save registers (SASS: LDG, 4 × F2F, LDG, …; a barrier between loads and sums did not hold them either), so the
// 16 loads ran one DRAM latency after the other: 100 µs for C5's 134 MB of partials (ncu: long-scoreboard stalls,
// 1.3 TB/s).
template <int CPT>
__global__ void __launch_bounds__(256) reduce_zp_kernel(const float* __restrict__ Zp, int64_t nrg, int64_t dpad, int mp,
                                                        int m, int64_t d, float* __restrict__ Z, int64_t ds) {
  pdl_enter();
  __shared__ float tr[128][65];
  extern __shared__ __align__(16) float4 stage[];    // [16][256]
  constexpr int GB = 16 / CPT;                       // partials per batch of loads
  const int tpc = mp >> 2;                           // threads per column (mp ≤ 128, multiple of 16)
  const int cpp = 256 / tpc;                         // columns per sweep of the block
  const int cpb = cpp * CPT;                         // columns per block (≤ 64)
  const int64_t x0 = (int64_t)blockIdx.x * cpb;
  const int xl = threadIdx.x / tpc, j4 = (threadIdx.x % tpc) * 4;
  double a[CPT][4];
#pragma unroll
  for (int cc = 0; cc < CPT; ++cc) a[cc][0] = a[cc][1] = a[cc][2] = a[cc][3] = 0.0;
  const int64_t gs = dpad * mp / 4;
  const uint32_t st0 = (uint32_t)__cvta_generic_to_shared(stage + threadIdx.x);
  for (int64_t g0 = 0; g0 < nrg; g0 += GB) {
    if (g0 > 0) __syncwarp();                        // (own slots only: no block barrier between batches)
#pragma unroll
    for (int cc = 0; cc < CPT; ++cc) {
      const int64_t x = min(x0 + xl + cc * cpp, d - 1);
      const float4* src = reinterpret_cast<const float4*>(Zp + x * mp + j4);
#pragma unroll
      for (int gg = 0; gg < GB; ++gg)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(st0 + (uint32_t)((cc * GB + gg) * 256 * 16)),
                     "l"(src + min(g0 + gg, nrg - 1) * gs)
                     : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
    for (int cc = 0; cc < CPT; ++cc) {
      const int64_t x = x0 + xl + cc * cpp;
#pragma unroll
      for (int gg = 0; gg < GB; ++gg)
        if (x < d && g0 + gg < nrg) {
          const float4 v = stage[(cc * GB + gg) * 256 + threadIdx.x];
          a[cc][0] += (double)v.x; a[cc][1] += (double)v.y;
          a[cc][2] += (double)v.z; a[cc][3] += (double)v.w;
        }
    }
  }
#pragma unroll
  for (int cc = 0; cc < CPT; ++cc) {
    const int c = xl + cc * cpp;
    tr[j4][c] = (float)a[cc][0]; tr[j4 + 1][c] = (float)a[cc][1];
    tr[j4 + 2][c] = (float)a[cc][2]; tr[j4 + 3][c] = (float)a[cc][3];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < m * cpb; e += 256) {
    const int j = e / cpb, c = e % cpb;
    if (x0 + c < d) Z[z_index(j, x0 + c, m, ds)] = tr[j][c];
  }
}

// The Z reduction of the power pass with the Gram of the CholQR that follows folded in (one rank, m ≤ 64, d-major
// Z): a CTA owns ZG_X = 2 features x and every component j.  Z is summed exactly as reduce_zp_cols_kernel sums
// it (sub-sum w over the row groups g ≡ w mod 8 in order, then the 8 sub-sums in w order: the same bits; 16
// loads in flight per thread — the sum is L2-latency bound, so it needs many CTAs and many loads in flight).
// The 8 CTAs of a cluster then gather their 16 rows of Z through distributed shared memory and each computes
// one eighth of the cluster's Gram partial Σ_x z_x z_xᵀ (fp64 of the stored fp32 values, x ascending) — one
// m×m partial per cluster, summed in cluster order by reduce_splits.  Replaces vec_gram's two launches on the
// Z the pass has just produced (15.8 + 1.9 µs for C3).
constexpr int ZG_X = 2, ZG_CL = 8, ZG_B = 4;
__global__ void __launch_bounds__(256) reduce_zp_gram_kernel(const float* __restrict__ Zp, int64_t nrg, int64_t dpad,
                                                             int mp, int m, int64_t d, float* __restrict__ Z,
                                                             double* __restrict__ Gpart) {
  pdl_enter();
  __shared__ double part[8][ZG_X * 64];
  __shared__ __align__(16) float zf[ZG_X * 64];
  __shared__ __align__(16) float zall[ZG_CL * ZG_X * 64];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t x0 = (int64_t)blockIdx.x * ZG_X;
  const int j0 = lane, j1 = lane + 32;
  double acc[ZG_X][2];
#pragma unroll
  for (int xi = 0; xi < ZG_X; ++xi) acc[xi][0] = acc[xi][1] = 0.0;
  const float* base[ZG_X];
#pragma unroll
  for (int xi = 0; xi < ZG_X; ++xi) base[xi] = Zp + min(x0 + xi, d - 1) * mp;
  const int64_t gstride = dpad * mp;
  // a batch's ZG_B·ZG_X·2 loads go through cp.async into the thread's own staging slots, one wait per batch: in
  // flight together by construction (as register loads ptxas kept runs of four and put the conversions of each run
  // behind it: four L2 round trips per batch instead of one)
  __shared__ float stg[ZG_B * ZG_X * 2][256];
  const uint32_t st0 = (uint32_t)__cvta_generic_to_shared(&stg[0][threadIdx.x]);
  const int jc0 = min(j0, m - 1), jc1 = min(j1, m - 1);
  for (int64_t g0 = warp; g0 < nrg; g0 += 8 * ZG_B) {
#pragma unroll
    for (int u = 0; u < ZG_B; ++u) {
      const int64_t g = g0 + 8 * u;
#pragma unroll
      for (int xi = 0; xi < ZG_X; ++xi) {
        const float* src = base[xi] + min(g, nrg - 1) * gstride;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(st0 + (uint32_t)(((u * ZG_X + xi) * 2) * 1024)),
                     "l"(src + jc0)
                     : "memory");
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(st0 + (uint32_t)(((u * ZG_X + xi) * 2 + 1) * 1024)),
                     "l"(src + jc1)
                     : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
    for (int u = 0; u < ZG_B; ++u)
      if (g0 + 8 * u < nrg) {
#pragma unroll
        for (int xi = 0; xi < ZG_X; ++xi) {
          acc[xi][0] += (double)(j0 < m ? stg[(u * ZG_X + xi) * 2][threadIdx.x] : 0.f);
          acc[xi][1] += (double)(j1 < m ? stg[(u * ZG_X + xi) * 2 + 1][threadIdx.x] : 0.f);
        }
      }
  }
#pragma unroll
  for (int xi = 0; xi < ZG_X; ++xi) {
    part[warp][xi * 64 + j0] = acc[xi][0];
    part[warp][xi * 64 + j1] = acc[xi][1];
  }
  __syncthreads();
  if (threadIdx.x < ZG_X * 64) {
    const int e = threadIdx.x, xi = e / 64, j = e % 64;
    const int64_t x = x0 + xi;
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += part[w][e];
    const float zv = (float)t;
    const bool live = x < d && j < m;
    zf[e] = live ? zv : 0.f;
    if (live) Z[(int64_t)j * d + x] = zv;
  }
  cluster_barrier();                             // every CTA's rows of Z are in its shared memory
  if (threadIdx.x < ZG_CL * ZG_X * 64 / 4) {       // gather the cluster's 16 rows (rank order = x order)
    const int r = threadIdx.x / (ZG_X * 16), o = threadIdx.x % (ZG_X * 16);
    uint32_t ra, a, b, c2, e2;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                 : "=r"(ra)
                 : "r"((uint32_t)__cvta_generic_to_shared(zf) + (uint32_t)o * 16u), "r"(r));
    asm volatile("ld.shared::cluster.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(a), "=r"(b), "=r"(c2), "=r"(e2) : "r"(ra));
    *reinterpret_cast<uint4*>(&zall[r * ZG_X * 64 + o * 4]) = make_uint4(a, b, c2, e2);
  }
  cluster_barrier();                             // every gather is done before any CTA may exit
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int mm = m * m, per = (mm + ZG_CL - 1) / ZG_CL;
  const int e0 = (int)rank * per, e1 = min(mm, e0 + per);
  double* out = Gpart + (int64_t)(blockIdx.x / ZG_CL) * mm;
  for (int e = e0 + threadIdx.x; e < e1; e += 256) {
    const int i = e / m, j = e % m;
    double t = 0.0;
#pragma unroll
    for (int x = 0; x < ZG_CL * ZG_X; ++x) t = fma((double)zall[x * 64 + i], (double)zall[x * 64 + j], t);
    out[e] = t;
  }
}

size_t zgram_part_bytes(int m, int64_t d) {
  return (size_t)ceil_div(ceil_div(d, (int64_t)ZG_X), (int64_t)ZG_CL) * m * m * sizeof(double);
}

// number of cluster partials reduce_zp_gram leaves (0: not applicable)
static int zgram_parts(int64_t nrg, int m, int64_t d, int64_t ds) {
  if (nrg <= 16 || m > 64 || ds != d) return 0;
  return (int)ceil_div(ceil_div(d, (int64_t)ZG_X), (int64_t)ZG_CL);
}

static void launch_reduce_zp(Ctx* c, const float* Zp, int64_t nrg, int64_t dpad, int mp, int m, int64_t d, float* Z) {
  const int64_t ds = c->z_block_cols > 0 ? c->z_block_cols : d;
  if (nrg > 16)
    launch_pdl(reduce_zp_cols_kernel, dim3(dim3((unsigned)d, (unsigned)ceil_div(m, 32))), dim3(256), 0, c->stream, Zp, nrg, dpad, mp, m, d, Z,
                                                                                            ds);
  else {
    const int cpp = 256 / (mp / 4);                  // columns per block sweep; CPT sweeps per block, ≤ 64 columns
    static const int cpt_cap = tune_env("PPCA_ZP_CPT", 4);
    const int cpt = std::min(std::min(nrg <= 4 ? 4 : (nrg <= 8 ? 2 : 1), std::max(1, 64 / cpp)), cpt_cap);
    const size_t stage = (size_t)16 * 256 * sizeof(float4);   // 64 KB + 33 KB static: two CTAs per SM
    static uint64_t attr = 0;
    if (first_on_device(&attr, c->device)) {
      cudaFuncSetAttribute(reduce_zp_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)stage);
      cudaFuncSetAttribute(reduce_zp_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)stage);
      cudaFuncSetAttribute(reduce_zp_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)stage);
    }
    if (cpt >= 4)
      launch_pdl(reduce_zp_kernel<4>, dim3((unsigned)ceil_div(d, (int64_t)(4 * cpp))), dim3(256), stage, c->stream, Zp, nrg, dpad, mp, m, d, Z, ds);
    else if (cpt >= 2)
      launch_pdl(reduce_zp_kernel<2>, dim3((unsigned)ceil_div(d, (int64_t)(2 * cpp))), dim3(256), stage, c->stream, Zp, nrg, dpad, mp, m, d, Z, ds);
    else
      launch_pdl(reduce_zp_kernel<1>, dim3((unsigned)ceil_div(d, (int64_t)cpp)), dim3(256), stage, c->stream, Zp, nrg, dpad, mp, m, d, Z, ds);
  }
}

// ============================================================================ host side
struct TcState {
  int sm = 148;
};

static int pad16(int m) { return (m + 15) & ~15; }

// one CTA per SM; one SM is left free while side-stream work (the Ritz solve of the previous
// iterate) may be resident, otherwise the CTA queued behind it delays the whole persistent pass
static int persistent_ctas(const Ctx* c) { return c->side_busy ? c->sm_count - 1 : c->sm_count; }

// How many 2-CTA clusters of a kernel (dynamic smem, threads) can be resident at once; cached per device in
// *cache.  The persistent pair kernels deal tiles statically, so a cluster beyond that number would start only
// when another has finished its whole share: launching more than fit would double the tail (a guard for
// partitioned GPUs and smem carve-outs; on a whole B200 all 74 pairs fit).
static int max_pair_clusters(Ctx* c, const void* kern, size_t smem, int threads, int* cache) {
  const int dev = c->device & 63;
  if (cache[dev] > 0) return cache[dev];
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(2 * (c->sm_count / 2)));
  cfg.blockDim = dim3((unsigned)threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n < 1) {
    cudaGetLastError();
    n = c->sm_count / 2;
  }
  cache[dev] = n;
  return n;
}

template <int MP, int XM>
static ppca_status launch_ka(Ctx* c, const CUtensorMap& tmW, const CUtensorMap& tmX, const CUtensorMap& tmXlo,
                             const KAParams& kp, int grid) {
  const size_t smem = ka::smem_bytes(MP, XM);
  auto kern = xw_tc_kernel<MP, XM>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<<<grid, ka::NTHREADS, smem, c->stream>>>(tmW, tmX, tmXlo, kp);
  PPCA_LAUNCH_CHECK(c, "xw_tc_kernel");
  return PPCA_OK;
}

template <int MP, bool XBF16, bool XLO, bool LEAN>
static ppca_status launch_kb(Ctx* c, const CUtensorMap& tmYT, const CUtensorMap& tmX, const CUtensorMap& tmXlo,
                             const KBParams& bp, int grid) {
  const size_t smem = kb::Cfg<MP, XLO, LEAN>::SMEM;
  auto kern = xty_tc_kernel<MP, XBF16, XLO, LEAN>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  launch_pdl(kern, dim3(grid), dim3(kb::NTHREADS), smem, c->stream, tmYT, tmX, tmXlo, bp);
  PPCA_LAUNCH_CHECK(c, "xty_tc_kernel");
  return PPCA_OK;
}

template <int MP, int XM, bool PAIR = false>
static ppca_status launch_ka2(Ctx* c, const CUtensorMap& tmW, const CUtensorMap& tmX, const CUtensorMap& tmXlo,
                              const KAParams& kp, int grid) {
  const size_t smem = ka2::Cfg<MP, XM, PAIR>::SMEM;
  auto kern = xw_tma_kernel<MP, XM, PAIR>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if constexpr (!PAIR) {
    launch_pdl(kern, dim3(grid), dim3(ka2::NTHREADS), smem, c->stream, tmW, tmX, tmXlo, kp);
  } else {                                          // CTA pairs: clusters of 2
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(ka2::NTHREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c->stream;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = g_pdl ? 2 : 1;
    cudaLaunchKernelEx(&cfg, kern, tmW, tmX, tmXlo, kp);
  }
  PPCA_LAUNCH_CHECK(c, "xw_tma_kernel");
  return PPCA_OK;
}

template <int XM>
static ppca_status dispatch_ka2(Ctx* c, int mp, const CUtensorMap& tmW, const CUtensorMap& tmX,
                                const CUtensorMap& tmXlo, const KAParams& kp, int grid) {
  switch (mp) {
    case 16: return launch_ka2<16, XM>(c, tmW, tmX, tmXlo, kp, grid);
    case 32: return launch_ka2<32, XM>(c, tmW, tmX, tmXlo, kp, grid);
    case 48: return launch_ka2<48, XM>(c, tmW, tmX, tmXlo, kp, grid);
    case 64: return launch_ka2<64, XM>(c, tmW, tmX, tmXlo, kp, grid);
    case 80: return launch_ka2<80, XM>(c, tmW, tmX, tmXlo, kp, grid);
    case 96: return launch_ka2<96, XM>(c, tmW, tmX, tmXlo, kp, grid);
    case 112: return launch_ka2<112, XM>(c, tmW, tmX, tmXlo, kp, grid);
    case 128: return launch_ka2<128, XM>(c, tmW, tmX, tmXlo, kp, grid);
  }
  return set_error(c, PPCA_ERR_UNSUPPORTED, "tcgen05 pass: m=%d unsupported", mp);
}

template <int XM>
static ppca_status dispatch_ka(Ctx* c, int mp, const CUtensorMap& tmW, const CUtensorMap& tmX,
                               const CUtensorMap& tmXlo, const KAParams& kp, int grid) {
  switch (mp) {
    case 16: return launch_ka<16, XM>(c, tmW, tmX, tmXlo, kp, grid);
    case 32: return launch_ka<32, XM>(c, tmW, tmX, tmXlo, kp, grid);
    case 48: return launch_ka<48, XM>(c, tmW, tmX, tmXlo, kp, grid);
    case 64: return launch_ka<64, XM>(c, tmW, tmX, tmXlo, kp, grid);
    case 80: return launch_ka<80, XM>(c, tmW, tmX, tmXlo, kp, grid);
    case 96: return launch_ka<96, XM>(c, tmW, tmX, tmXlo, kp, grid);
    case 112: return launch_ka<112, XM>(c, tmW, tmX, tmXlo, kp, grid);
    case 128: return launch_ka<128, XM>(c, tmW, tmX, tmXlo, kp, grid);
  }
  return set_error(c, PPCA_ERR_UNSUPPORTED, "tcgen05 pass: m=%d unsupported", mp);
}

template <bool XBF16, bool XLO, bool LEAN = false>
static ppca_status dispatch_kb(Ctx* c, int mp, const CUtensorMap& tmYT, const CUtensorMap& tmX,
                               const CUtensorMap& tmXlo, const KBParams& bp, int grid) {
  switch (mp) {
    case 16: return launch_kb<16, XBF16, XLO, LEAN>(c, tmYT, tmX, tmXlo, bp, grid);
    case 32: return launch_kb<32, XBF16, XLO, LEAN>(c, tmYT, tmX, tmXlo, bp, grid);
    case 48: return launch_kb<48, XBF16, XLO, LEAN>(c, tmYT, tmX, tmXlo, bp, grid);
    case 64: return launch_kb<64, XBF16, XLO, LEAN>(c, tmYT, tmX, tmXlo, bp, grid);
    case 80: return launch_kb<80, XBF16, XLO, LEAN>(c, tmYT, tmX, tmXlo, bp, grid);
    case 96: return launch_kb<96, XBF16, XLO, LEAN>(c, tmYT, tmX, tmXlo, bp, grid);
    case 112: return launch_kb<112, XBF16, XLO, LEAN>(c, tmYT, tmX, tmXlo, bp, grid);
    case 128: return launch_kb<128, XBF16, XLO, LEAN>(c, tmYT, tmX, tmXlo, bp, grid);
  }
  return set_error(c, PPCA_ERR_UNSUPPORTED, "tcgen05 pass: m=%d unsupported", mp);
}

// TMA maps of X's bf16 planes (box 64 columns × box_rows rows): bf16 X → tmX; split → tmX = hi plane,
// tmXlo = lo plane (the row stride of a split row is 4·ld bytes = 2·ld bf16)
static bool make_x_maps(const ppca_matrix* X, uint32_t box_rows, CUtensorMap* hi, CUtensorMap* lo) {
  if (X->dtype == PPCA_BF16) return make_map_bf16(hi, X->data, X->d, X->n_local, X->ld, box_rows);
  const __nv_bfloat16* base = static_cast<const __nv_bfloat16*>(X->data);
  return make_map_bf16(hi, base, X->d, X->n_local, 2 * X->ld, box_rows) &&
         make_map_bf16(lo, base + X->d, X->d, X->n_local, 2 * X->ld, box_rows);
}

ppca_status pass_tc_prepare(Ctx* c, const ppca_matrix* X, int m, PassPlan* plan) {
  if (!encode_fn()) return set_error(c, PPCA_ERR_UNSUPPORTED, "cuTensorMapEncodeTiled unavailable");
  if (X->d % 8 != 0 || X->d < 64) return set_error(c, PPCA_ERR_UNSUPPORTED, "tcgen05 pass needs d %% 8 == 0, d >= 64");
  if (m > 128 || m < 1) return set_error(c, PPCA_ERR_UNSUPPORTED, "tcgen05 pass needs m <= 128");
  if (X->n_local < 1) return set_error(c, PPCA_ERR_UNSUPPORTED, "tcgen05 pass needs >= 1 local row");
  if (reinterpret_cast<uintptr_t>(X->data) % 16) return set_error(c, PPCA_ERR_UNSUPPORTED, "X not 16B aligned");
  if (X->n_local < 128) {
    // a short shard or minibatch window (the last block of a schedule): one partial tile whose rows beyond
    // n_local the TMA fills with zeros — if the driver accepts a 128-row box over fewer rows
    CUtensorMap probe, probe_lo;
    if (X->dtype == PPCA_F32 || !make_x_maps(X, 128, &probe, &probe_lo))
      return set_error(c, PPCA_ERR_UNSUPPORTED, "tcgen05 pass: %lld rows do not fill a TMA tile", (long long)X->n_local);
  }
  plan->impl = 2;
  return PPCA_OK;
}

// W' (bf16 + its fp32 value copy) → S_TC1;  returns pointers
static ppca_status prep_w(Ctx* c, const float* W, int m, int mp, int64_t d, __nv_bfloat16** Wb, float** Wr) {
  if (c->wprep_for == W && W) {                   // CholQR's apply wrote this W's operand already
    *Wb = c->wprep_b;
    *Wr = c->wprep_r;
    c->wprep_for = nullptr;
    return PPCA_OK;
  }
  uint8_t* buf = (uint8_t*)scratch(c, S_TC1, (size_t)2 * mp * d * 2 + (size_t)m * d * 4 + 256);
  if (!buf) return set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
  *Wb = reinterpret_cast<__nv_bfloat16*>(buf);
  *Wr = reinterpret_cast<float*>(buf + (((size_t)2 * mp * d * 2 + 255) & ~(size_t)255));
  launch_pdl(prep_w_kernel, dim3((unsigned)ceil_div((int64_t)mp * d, 1024)), dim3(256), 0, c->stream, W, m, mp, d, *Wb, *Wr);
  PPCA_LAUNCH_CHECK(c, "prep_w");
  return PPCA_OK;
}

static ppca_status run_ka(Ctx* c, const ppca_matrix* X, const __nv_bfloat16* Wb, int m, int mp, double* S,
                          __nv_bfloat16* YT, int64_t ldyt, int ksplit = 1, float* Ypart = nullptr,
                          const int32_t* tiles = nullptr, int64_t ntiles_sel = -1) {
  // kernel A2 on CTA pairs (2-CTA UMMA, W' split across the pair): bf16 X with m padded to 128 (C5), whole
  // tiles; PPCA_A2_PAIR=0 disables
  static int pair_env = -1;
  if (pair_env < 0) pair_env = tune_env("PPCA_A2_PAIR", 1);
  const bool pair = pair_env && X->dtype == PPCA_BF16 && mp == 128 && ksplit == 1 && tiles == nullptr &&
                    persistent_ctas(c) >= 2;
  CUtensorMap tmW, tmX, tmXlo;
  if (!make_map_bf16(&tmW, Wb, X->d, 2 * mp, X->d, pair ? mp : 2 * mp))
    return set_error(c, PPCA_ERR_CUDA, "tensor map W failed");
  tmX = tmXlo = tmW;   // unused unless X is staged by TMA
  if (X->dtype != PPCA_F32 && !make_x_maps(X, 128, &tmX, &tmXlo)) return set_error(c, PPCA_ERR_CUDA, "tensor map X failed");
  KAParams kp;
  kp.X = X->data; kp.n = X->n_local; kp.d = X->d; kp.ld = X->ld; kp.m = m; kp.mp = mp;
  kp.ntiles = tiles ? ntiles_sel : ceil_div(X->n_local, ka::BM);
  kp.tiles = tiles;
  kp.nk = ceil_div(X->d, ka::BK);
  kp.YT = YT; kp.ldyt = ldyt;
  kp.ksplit = ksplit;
  kp.kper = ceil_div(kp.nk, (int64_t)ksplit);
  kp.Ypart = Ypart;
  static int dbg = -1;
  if (dbg < 0) dbg = tune_env("PPCA_DBG", 0);
  kp.dbg = dbg;
  int grid = (int)std::max<int64_t>(1, std::min<int64_t>(persistent_ctas(c), kp.ntiles * ksplit));
  if (pair) {
    static int cache[64] = {};
    const int maxc = max_pair_clusters(c, (const void*)xw_tma_kernel<128, 1, true>, ka2::Cfg<128, 1, true>::SMEM,
                                       ka2::NTHREADS, cache);
    grid = (int)std::max<int64_t>(2, std::min<int64_t>(std::min(persistent_ctas(c) & ~1, 2 * maxc),
                                                       2 * ((kp.ntiles + 1) / 2)));
  }
  // TMA-staged X (bf16, split) runs kernel A2; its S partial has 2·mp rows when S is on the tensor cores
  const bool tma_x = X->dtype != PPCA_F32;
  const bool smma = tma_x && mp == 64;
  double* Spart = (double*)scratch(c, S_TC0, (size_t)grid * (smma ? 2 : 1) * mp * mp * sizeof(double));
  if (!Spart) return set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
  kp.Spart = Spart;
  kernel_timer_mark(c, 0);
  PPCA_TRY(pair                          ? (launch_ka2<128, 1, true>(c, tmW, tmX, tmXlo, kp, grid))
           : X->dtype == PPCA_BF16        ? dispatch_ka2<1>(c, mp, tmW, tmX, tmXlo, kp, grid)
           : X->dtype == PPCA_F32_SPLIT ? dispatch_ka2<2>(c, mp, tmW, tmX, tmXlo, kp, grid)
                                        : dispatch_ka<0>(c, mp, tmW, tmX, tmXlo, kp, grid));
  kernel_timer_mark(c, 0);
  if (ksplit > 1) return PPCA_OK;                 // partial Y out; the caller forms S from the summed Y
  if (smma)
    launch_pdl(reduce_spart2_kernel, dim3((unsigned)ceil_div(m * m, 32)), dim3(256), 0, c->stream, Spart, grid, mp, m, S);
  else
    launch_pdl(reduce_spart_kernel, dim3((unsigned)ceil_div(m * m, 32)), dim3(256), 0, c->stream, Spart, grid, mp, m, S);
  PPCA_LAUNCH_CHECK(c, "reduce_spart");
  return PPCA_OK;
}

// Y of a K-split row window and S = YᵀY in one pass over the partials: block = YS_RB rows.  Y = Σ_parts Ypart
// in part order (fp32), written as the Yᵀ bf16 pair [Y_hi; Y_lo] [2·mp][ldyt] (rows ≥ n zero) for kernel B;
// the block's rows also give a partial S_b = Σ_rows y yᵀ (fp64 products and sums, 4×4 register tiles per
// thread) that launch_reduce_splits_f64 sums in block order.
constexpr int YS_RB = 32;
static size_t ysum_s_smem(int mp) {
  const size_t rows = (size_t)YS_RB * (mp + 1);
  return ((rows + 3) & ~(size_t)3) * sizeof(float) + (size_t)16 * 256 * sizeof(float) + rows * sizeof(double);
}

__global__ void __launch_bounds__(256) ysum_s_kernel(const float* __restrict__ Ypart, int ksplit, int64_t n, int mp,
                                                     int m, __nv_bfloat16* __restrict__ YT, int64_t ldyt,
                                                     double* __restrict__ Spart) {
  pdl_enter();
  // YS_RB × (mp + 1) floats (the Y rows), [16][256] floats of load staging, YS_RB × (mp + 1) doubles (the same
  // rows for the S tiles: one conversion per element instead of eight per 16 DFMA)
  extern __shared__ __align__(16) float ysm[];
  const int ld = mp + 1;
  float* stg = ysm + ((YS_RB * ld + 3) & ~3);
  double* ysd = reinterpret_cast<double*>(stg + 16 * 256);
  const int64_t r0 = (int64_t)blockIdx.x * YS_RB;
  const int cnt = YS_RB * mp;
  const uint32_t st0 = (uint32_t)__cvta_generic_to_shared(stg + threadIdx.x);
  for (int e0 = threadIdx.x; e0 < cnt; e0 += 4 * 256) {
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int q0 = 0; q0 < ksplit; q0 += 4) {
      // 4 parts × 4 elements: 16 cp.async into the thread's own staging slots and one wait — in flight together by
      // construction (as register loads the compiler put every add right behind its load: 16 L2 round trips in a
      // row, the reason this kernel took 14 µs on C4; clamped addresses, masked at the sum)
#pragma unroll
      for (int qq = 0; qq < 4; ++qq)
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int e = min(e0 + u * 256, cnt - 1);
          const int64_t r = min(r0 + e / mp, n - 1);
          const float* src = Ypart + ((int64_t)min(q0 + qq, ksplit - 1) * n + r) * mp + e % mp;
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(st0 + (uint32_t)((qq * 4 + u) * 256 * 4)), "l"(src)
                       : "memory");
        }
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
      for (int qq = 0; qq < 4; ++qq)
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int e = e0 + u * 256;
          const bool ok = q0 + qq < ksplit && e < cnt && r0 + e / mp < n;
          acc[u] += ok ? stg[(qq * 4 + u) * 256 + threadIdx.x] : 0.f;   // part order unchanged
        }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + u * 256;
      if (e < cnt) {
        ysm[(e / mp) * ld + e % mp] = acc[u];
        ysd[(e / mp) * ld + e % mp] = (double)acc[u];
      }
    }
  }
  __syncthreads();
  // the Yᵀ pair (rows < ldyt; rows ≥ n are zero)
  for (int e = threadIdx.x; e < mp * YS_RB; e += 256) {
    const int j = e / YS_RB, rr = e % YS_RB;
    if (r0 + rr < ldyt) {
      const float y = ysm[rr * ld + j];
      const __nv_bfloat16 hi = __float2bfloat16_rn(y);
      YT[(int64_t)j * ldyt + r0 + rr] = hi;
      YT[(int64_t)(mp + j) * ldyt + r0 + rr] = __float2bfloat16_rn(y - __bfloat162float(hi));
    }
  }
  // partial S of the block's rows
  const int nt4 = mp / 4;
  double* Sb = Spart + (int64_t)blockIdx.x * m * m;
  for (int tile = threadIdx.x; tile < nt4 * nt4; tile += 256) {
    const int bi = tile / nt4, bj = tile % nt4;
    double a[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) a[u][v] = 0.0;
    for (int rr = 0; rr < YS_RB; ++rr) {
      const double* row = ysd + rr * ld;
      double yi[4], yj[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        yi[u] = row[bi * 4 + u];
        yj[u] = row[bj * 4 + u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) a[u][v] = fma(yi[u], yj[v], a[u][v]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int i = bi * 4 + u, j = bj * 4 + v;
        if (i < m && j < m) Sb[i * m + j] = a[u][v];
      }
  }
}

static int pick_ksplit_tiles(const Ctx* c, const ppca_matrix* X, int64_t ntiles, int64_t nk);

// K split for short row windows (a minibatch step): enough (tile, K part) items to cover the SMs
static int pick_ksplit(const Ctx* c, const ppca_matrix* X, int64_t nk) {
  return pick_ksplit_tiles(c, X, ceil_div(X->n_local, ka::BM), nk);
}

static int pick_ksplit_tiles(const Ctx* c, const ppca_matrix* X, int64_t ntiles, int64_t nk) {
  if (X->dtype == PPCA_F32) return 1;                 // the converter kernel A has no K split
  const int64_t ctas = persistent_ctas(c);
  if (2 * ntiles > ctas) return 1;
  int64_t ks = std::min<int64_t>(nk, std::max<int64_t>(1, ctas / ntiles));
  const int64_t kper = ceil_div(nk, ks);
  return (int)ceil_div(nk, kper);
}

// refine-mode pass (S only).  Fewer row tiles than SMs (huge d with few rows, a row-tile sample): K split
// over the SMs, the fp32 partial Y of each K part summed in part order, S from the sum (ysum_s)
ppca_status pass_tc_gram(Ctx* c, const ppca_matrix* X, const PassPlan* plan, const float* W, int m, double* S) {
  const int mp = pad16(m);
  __nv_bfloat16* Wb;
  float* Wr;
  PPCA_TRY(prep_w(c, W, m, mp, X->d, &Wb, &Wr));
  const_cast<PassPlan*>(plan)->Wop = Wr;
  const int64_t n = X->n_local;
  const int64_t ntiles = plan->tiles_dev ? plan->ntiles_sel : ceil_div(n, ka::BM);
  const int ksplit = ntiles > 0 ? pick_ksplit_tiles(c, X, ntiles, ceil_div(X->d, ka::BK)) : 1;
  if (ksplit == 1) return run_ka(c, X, Wb, m, mp, S, nullptr, 0, 1, nullptr, plan->tiles_dev, plan->ntiles_sel);
  float* Ypart = (float*)scratch(c, S_TC3, (size_t)ksplit * n * mp * sizeof(float));
  const int64_t nb = ceil_div(n, (int64_t)YS_RB);
  double* Sp = (double*)scratch(c, S_NTSTAGE, (size_t)nb * m * m * sizeof(double));
  if (!Ypart || !Sp) return set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
  if (plan->tiles_dev)                          // rows outside the sample stay zero in every part
    PPCA_TRY(check_cuda(c, cudaMemsetAsync(Ypart, 0, (size_t)ksplit * n * mp * sizeof(float), c->stream), "zero Y"));
  PPCA_TRY(run_ka(c, X, Wb, m, mp, S, nullptr, 0, ksplit, Ypart, plan->tiles_dev, plan->ntiles_sel));
  launch_pdl(ysum_s_kernel, dim3((unsigned)nb), dim3(256), ysum_s_smem(mp), c->stream, Ypart, ksplit, n, mp, m,
                                                                                            nullptr, 0, Sp);
  PPCA_LAUNCH_CHECK(c, "ysum_s");
  return launch_reduce_splits_f64(c, Sp, (int)nb, (int64_t)m * m, S);
}


template <int XM, int NSTA, int NWS, int NSTB>
static constexpr size_t fused_smem() {
  return 1024 + (size_t)NSTA * (XM == 2 ? 2 * kf::XPL : kf::XPL) + (size_t)NWS * kf::WST +
         (size_t)NSTB * (kf::BX + kf::BY) + 256;
}

// The CTAs of a row group wait on each other's tile flags, so the grid must be co-resident: a cooperative
// launch guarantees it or fails (cudaErrorCooperativeLaunchTooLarge: fewer free SMs than CTAs, e.g. under an
// MPS / green-context partition), in which case the caller runs the two-kernel pass instead.
template <int XM, int NSTA, int NWS, int NSTB>
static cudaError_t launch_fused(Ctx* c, int grid, const CUtensorMap& tmW, const CUtensorMap& tmX,
                                const CUtensorMap& tmXlo, const CUtensorMap& tmXb, const CUtensorMap& tmY,
                                const KFParams& fp) {
  constexpr size_t smem = fused_smem<XM, NSTA, NWS, NSTB>();
  static_assert(smem <= 227 * 1024, "fused kernel shared memory budget");
  auto kern = xwz_fused_kernel<XM, NSTA, NWS, NSTB>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kf::NTHREADS, smem) != cudaSuccess ||
      per_sm * c->sm_count < grid) {
    cudaGetLastError();
    return cudaErrorCooperativeLaunchTooLarge;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kf::NTHREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, tmW, tmX, tmXlo, tmXb, tmY, fp);
}

template <int XM>
static cudaError_t launch_fused_cfg(Ctx* c, int cfg, int grid, const CUtensorMap& tmW, const CUtensorMap& tmX,
                                    const CUtensorMap& tmXlo, const CUtensorMap& tmXb, const CUtensorMap& tmY,
                                    const KFParams& fp) {
  // (X stages, W' stages, B stages of KR = 64 rows).  Measured on C3, one box: 32-row B stages (2,2,5)
  // 1.088 ms -> 64-row B stages (2,2,2) 0.951 ms, (3,2,2) 0.993, (2,1,3) 1.018 (larger TMA boxes and half
  // the B-stream barrier round trips); PPCA_FUSED_CFG (experiment builds) selects the others
  switch (cfg) {
    case 6: return launch_fused<XM, 3, 2, 2>(c, grid, tmW, tmX, tmXlo, tmXb, tmY, fp);
    case 7: return launch_fused<XM, 2, 1, 3>(c, grid, tmW, tmX, tmXlo, tmXb, tmY, fp);
    default: return launch_fused<XM, 2, 2, 2>(c, grid, tmW, tmX, tmXlo, tmXb, tmY, fp);
  }
}

// The single-read power pass: TMA-staged X (bf16 / split), m ≤ 64 (padded to 64), d ≤ KSEG·BK (one
// accumulation segment), a whole row tile per CTA at least.
static bool fused_eligible(const Ctx* c, const ppca_matrix* X, int mp, bool precise) {
  return (c->pass_impl == 0 || c->pass_impl == 2 || c->pass_impl == 4) && !precise && X->dtype != PPCA_F32 && mp == 64 &&
         X->d <= ka2::KSEG * ka2::BK &&
         X->n_local >= 128;
}

// *launched = false (status OK) when the grid cannot be co-resident: the caller runs the two-kernel pass.
static ppca_status pass_fused_power(Ctx* c, const ppca_matrix* X, const __nv_bfloat16* Wb, int m, float* Z,
                                    double* S, bool* launched) {
  *launched = false;
  const int mp = 64;
  const int64_t n = X->n_local, d = X->d;
  const int64_t ntiles = ceil_div(n, kf::BM);
  const int64_t ctas = persistent_ctas(c);
  const int ndg = (int)ceil_div(d, (int64_t)kf::DG);
  int nrg = (int)std::max<int64_t>(1, std::min<int64_t>(ctas / ndg, ntiles));
  const int64_t tpr = ceil_div(ntiles, (int64_t)nrg);
  nrg = (int)ceil_div(ntiles, tpr);
  const int grid = ndg * nrg;
  const int64_t nrow_pad = ntiles * kf::BM;
  __nv_bfloat16* Yrm = (__nv_bfloat16*)scratch(c, S_Y, (size_t)nrow_pad * 2 * mp * 2);
  double* Spart = (double*)scratch(c, S_TC0, (size_t)grid * 2 * mp * mp * sizeof(double));
  const int64_t dpad = (int64_t)ndg * kf::DG;
  float* Zp = (float*)scratch(c, S_PART, (size_t)nrg * dpad * mp * sizeof(float));
  if (!Yrm || !Spart || !Zp) return set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
  if (c->flags_n < ntiles) {                     // per-tile ready flags: zeroed once, epochs count up
    if (c->flags) {
      cudaStreamSynchronize(c->stream);
      cudaFree(c->flags);
      c->flags = nullptr;
    }
    if (cudaMalloc(&c->flags, (size_t)ntiles * sizeof(int)) != cudaSuccess) {
      cudaGetLastError();
      c->flags_n = 0;
      return set_error(c, PPCA_ERR_CUDA, "flags alloc failed");
    }
    PPCA_TRY(check_cuda(c, cudaMemsetAsync(c->flags, 0, (size_t)ntiles * sizeof(int), c->stream), "flags"));
    c->flags_n = ntiles;
    c->epoch = 0;
  }
  if (++c->epoch >= (1 << 30)) {
    PPCA_TRY(check_cuda(c, cudaMemsetAsync(c->flags, 0, (size_t)c->flags_n * sizeof(int), c->stream), "flags"));
    c->epoch = 1;
  }
  CUtensorMap tmW, tmX, tmXlo, tmXb, tmXblo, tmY;
  if (!make_map_bf16(&tmW, Wb, d, 2 * mp, d, 2 * mp)) return set_error(c, PPCA_ERR_CUDA, "tensor map W failed");
  tmXlo = tmW;
  if (!make_x_maps(X, kf::BM, &tmX, &tmXlo) || !make_x_maps(X, kf::KR, &tmXb, &tmXblo))
    return set_error(c, PPCA_ERR_CUDA, "tensor map X failed");
  if (!make_map_bf16(&tmY, Yrm, 2 * mp, nrow_pad, 2 * mp, kf::KR)) return set_error(c, PPCA_ERR_CUDA, "tensor map Y failed");
  KFParams fp;
  fp.n = n; fp.d = d; fp.m = m;
  fp.ntiles = ntiles; fp.nk = ceil_div(d, (int64_t)kf::BK); fp.nseg = 1;
  fp.ndg = ndg; fp.nrg = nrg; fp.tiles_per_rg = tpr;
  fp.Yrm = Yrm; fp.nrow_pad = nrow_pad; fp.Spart = Spart; fp.Zp = Zp;
  fp.flags = c->flags; fp.epoch = c->epoch;
  static int pf = -1;
  if (pf < 0) pf = tune_env("PPCA_FUSED_PF", 0);
  fp.pf = pf;
  static int dbg = -1;
  if (dbg < 0) dbg = tune_env("PPCA_DBG", 0);
  fp.dbg = dbg;
  static int hip = -1;
  if (hip < 0) hip = tune_env("PPCA_FUSED_HI", 0);
  fp.hi_policy = hip;
  static int lag = -1;
  // A-stream lead over the B-stream capped at 2 rounds (measured on C3: dram reads 5.73 → 5.41 GB, pass
  // −1.6 %; 1 round starves the overlap, 3 = unbounded); PPCA_FUSED_LAG overrides (0 = off)
  if (lag < 0) lag = tune_env("PPCA_FUSED_LAG", 2);
  fp.lag = lag;
  fp.err = c->d_err;
  if (c->s_defer) cudaStreamWaitEvent(c->stream, c->s_ev_red, 0);   // the previous S partials were reduced
  kernel_timer_mark(c, 0);
  static int cfg = -1;
  if (cfg < 0) cfg = tune_env("PPCA_FUSED_CFG", 0);
  const cudaError_t le = X->dtype == PPCA_F32_SPLIT ? launch_fused_cfg<2>(c, cfg, grid, tmW, tmX, tmXlo, tmXb, tmY, fp)
                                                    : launch_fused_cfg<1>(c, cfg, grid, tmW, tmX, tmXlo, tmXb, tmY, fp);
  if (le == cudaErrorCooperativeLaunchTooLarge) {   // not co-resident here: nothing was launched
    cudaGetLastError();
    if (c->timing && c->kev_used[0] > 0) c->kev_used[0]--;   // drop the unmatched timer mark
    return PPCA_OK;
  }
  if (le != cudaSuccess) return check_cuda(c, le, "xwz_fused_kernel");
  PPCA_LAUNCH_CHECK(c, "xwz_fused_kernel");
  kernel_timer_mark(c, 0);
  *launched = true;
  if (c->s_skip) {                                // the caller does not use S (power priming without θ history)
  } else if (c->s_defer) {                        // S is reduced later, on the stream that consumes it
    cudaEventRecord(c->s_ev_pass, c->stream);
    c->s_pending = true;
    c->s_part = Spart;
    c->s_parts = grid;
    c->s_mp = mp;
    c->s_m = m;
  } else {
    launch_pdl(reduce_spart2_kernel, dim3((unsigned)ceil_div(m * m, 32)), dim3(256), 0, c->stream, Spart, grid, mp, m, S);
    PPCA_LAUNCH_CHECK(c, "reduce_spart");
  }
  launch_reduce_zp(c, Zp, nrg, dpad, mp, m, d, Z);
  PPCA_LAUNCH_CHECK(c, "reduce_zp");
  return PPCA_OK;
}

// ============================================================================ d-sliced pair pass (tc_pair.cuh)
template <int XM, int NSTA, int NWS, int NSTB, int KR>
static constexpr size_t pair_smem() {
  return 1024 + (size_t)NSTA * (XM == 2 ? 2 * kp2::XPL : kp2::XPL) + (size_t)NWS * kp2::WST +
         (size_t)NSTB * kp2::NCH * KR * 128 + 2 * kp2::YSL + 256;
}

// Clusters of 2 (a pair's waits never leave the cluster, which is co-scheduled by construction)
template <int XM, int NSTA, int NWS, int NSTB, int KR>
static cudaError_t launch_pair(Ctx* c, int grid, const CUtensorMap& tmW, const CUtensorMap& tmX,
                               const CUtensorMap& tmXlo, const CUtensorMap& tmXb, const KP2Params& pp) {
  constexpr size_t smem = pair_smem<XM, NSTA, NWS, NSTB, KR>();
  static_assert(smem <= 227 * 1024, "pair kernel shared memory budget");
  auto kern = xwz_pair_kernel<XM, NSTA, NWS, NSTB, KR>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kp2::NTHREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // its prologue overlaps prep_w's tail
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = g_pdl ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kern, tmW, tmX, tmXlo, tmXb, pp);
}

template <int XM, int NSTA, int NWS, int NSTB, int KR>
static int pair_max_clusters(Ctx* c) {
  static int cache[64] = {};
  return max_pair_clusters(c, (const void*)xwz_pair_kernel<XM, NSTA, NWS, NSTB, KR>,
                           pair_smem<XM, NSTA, NWS, NSTB, KR>(), kp2::NTHREADS, cache);
}

template <int XM>
static int pair_max_clusters_cfg(Ctx* c, int cfg) {
  switch (cfg) {
    case 1: return pair_max_clusters<XM, 2, 2, 2, 32>(c);
    case 2: return pair_max_clusters<XM, 2, 2, 3, 16>(c);
    case 3: return pair_max_clusters<XM, 2, 3, 3, 16>(c);
    case 4: return pair_max_clusters<XM, 3, 1, 3, 16>(c);
    case 5: return pair_max_clusters<XM, 2, 2, 4, 16>(c);
    default: return pair_max_clusters<XM, 3, 2, 2, 16>(c);
  }
}

template <int XM>
static cudaError_t launch_pair_cfg(Ctx* c, int cfg, int grid, const CUtensorMap& tmW, const CUtensorMap& tmX,
                                   const CUtensorMap& tmXlo, const CUtensorMap& tmXb, const KP2Params& pp) {
  // (X stages, W' stages, B stages, rows per B stage); PPCA_PAIR_CFG (experiment builds) selects the others
  switch (cfg) {
    case 1: return launch_pair<XM, 2, 2, 2, 32>(c, grid, tmW, tmX, tmXlo, tmXb, pp);
    case 2: return launch_pair<XM, 2, 2, 3, 16>(c, grid, tmW, tmX, tmXlo, tmXb, pp);
    case 3: return launch_pair<XM, 2, 3, 3, 16>(c, grid, tmW, tmX, tmXlo, tmXb, pp);
    case 4: return launch_pair<XM, 3, 1, 3, 16>(c, grid, tmW, tmX, tmXlo, tmXb, pp);
    case 5: return launch_pair<XM, 2, 2, 4, 16>(c, grid, tmW, tmX, tmXlo, tmXb, pp);
    default: return launch_pair<XM, 3, 2, 2, 16>(c, grid, tmW, tmX, tmXlo, tmXb, pp);
  }
}

// The d-sliced pair pass: TMA-staged X (bf16 / split), m ≤ 64 (padded to 64), SL < d ≤ 2·SL, whole tiles.
static bool pair_eligible(const Ctx* c, const ppca_matrix* X, int mp, bool precise) {
  return (c->pass_impl == 0 || c->pass_impl == 2) && !precise && X->dtype != PPCA_F32 && mp == 64 &&
         X->d > kp2::SL && X->d <= 2 * kp2::SL && X->n_local >= 128 && persistent_ctas(c) >= 2;
}

static ppca_status pass_pair_power(Ctx* c, const ppca_matrix* X, const __nv_bfloat16* Wb, int m, float* Z, double* S) {
  const int mp = 64;
  const int64_t n = X->n_local, d = X->d;
  const int64_t ntiles = ceil_div(n, kp2::BM);
  static int cfg = -1;
  if (cfg < 0) cfg = tune_env("PPCA_PAIR_CFG", 0);
  const int maxc = X->dtype == PPCA_F32_SPLIT ? pair_max_clusters_cfg<2>(c, cfg) : pair_max_clusters_cfg<1>(c, cfg);
  static int nrg_cap = -1;                        // PPCA_PAIR_NRG (experiment builds): cap the cluster count
  if (nrg_cap < 0) nrg_cap = tune_env("PPCA_PAIR_NRG", 0);
  int nrg = (int)std::max<int64_t>(1, std::min<int64_t>(std::min(persistent_ctas(c) / 2, maxc), ntiles));
  if (nrg_cap > 0) nrg = std::min(nrg, nrg_cap);
  const int64_t tpr = ceil_div(ntiles, (int64_t)nrg);
  nrg = (int)ceil_div(ntiles, tpr);
  const int grid = 2 * nrg;
  double* Spart = (double*)scratch(c, S_TC0, (size_t)grid * 2 * mp * mp * sizeof(double));
  const int64_t dpad = 2 * kp2::SL;
  float* Zp = (float*)scratch(c, S_PART, (size_t)nrg * dpad * mp * sizeof(float));
  if (!Spart || !Zp) return set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
  CUtensorMap tmW, tmX, tmXlo, tmXb, tmXblo;
  if (!make_map_bf16(&tmW, Wb, d, 2 * mp, d, 2 * mp)) return set_error(c, PPCA_ERR_CUDA, "tensor map W failed");
  tmXlo = tmW;
  const uint32_t kr = (cfg == 1) ? 32 : 16;
  if (!make_x_maps(X, kp2::BM, &tmX, &tmXlo) || !make_x_maps(X, kr, &tmXb, &tmXblo))
    return set_error(c, PPCA_ERR_CUDA, "tensor map X failed");
  KP2Params pp;
  pp.n = n; pp.d = d; pp.ntiles = ntiles; pp.nrg = nrg; pp.tiles_per_rg = tpr;
  pp.Spart = Spart; pp.Zp = Zp; pp.trace = nullptr;
  static const int pair_pol = tune_env("PPCA_PAIR_POL", 0 | 2 << 2 | 2 << 4);   // hi evict_last, lo / re-read evict_first
  pp.pol = pair_pol;
#ifdef PPCA_EXPERIMENTS
  static int trace_at = -1, launches = 0;         // PPCA_TRACE=k: stamp the k-th launch, dump it to gpurun_out/
  if (trace_at < 0) trace_at = tune_env("PPCA_TRACE", 0);
  static long long* tbuf = nullptr;
  const size_t tbytes = ((size_t)2 * KP2_TRACE_TILES * KP2_TRACE_EV + 2 * 1024) * sizeof(long long);
  const bool tracing = trace_at > 0 && ++launches == trace_at;
  if (tracing) {
    if (!tbuf) cudaMalloc(&tbuf, tbytes);
    cudaMemsetAsync(tbuf, 0, tbytes, c->stream);
    pp.trace = tbuf;
  }
#endif
  if (c->s_defer) cudaStreamWaitEvent(c->stream, c->s_ev_red, 0);   // the previous S partials were reduced
  kernel_timer_mark(c, 0);
  const cudaError_t le = X->dtype == PPCA_F32_SPLIT ? launch_pair_cfg<2>(c, cfg, grid, tmW, tmX, tmXlo, tmXb, pp)
                                                    : launch_pair_cfg<1>(c, cfg, grid, tmW, tmX, tmXlo, tmXb, pp);
  if (le != cudaSuccess) return check_cuda(c, le, "xwz_pair_kernel");
  PPCA_LAUNCH_CHECK(c, "xwz_pair_kernel");
#ifdef PPCA_EXPERIMENTS
  if (tracing) {
    std::vector<long long> hbuf(tbytes / sizeof(long long));
    cudaMemcpyAsync(hbuf.data(), tbuf, tbytes, cudaMemcpyDeviceToHost, c->stream);
    cudaStreamSynchronize(c->stream);
    if (FILE* f = fopen("gpurun_out/pair_trace.bin", "wb")) {
      fwrite(hbuf.data(), 1, tbytes, f);
      fclose(f);
    }
  }
#endif
  kernel_timer_mark(c, 0);
  if (c->s_skip) {                                // the caller does not use S (power priming without θ history)
  } else if (c->s_defer) {                        // S is reduced later, on the stream that consumes it
    cudaEventRecord(c->s_ev_pass, c->stream);
    c->s_pending = true;
    c->s_part = Spart;
    c->s_parts = grid;
    c->s_mp = mp;
    c->s_m = m;
  } else {
    launch_pdl(reduce_spart2_kernel, dim3((unsigned)ceil_div(m * m, 32)), dim3(256), 0, c->stream, Spart, grid, mp, m, S);
    PPCA_LAUNCH_CHECK(c, "reduce_spart");
  }
  const int ngp = c->zgram_want ? zgram_parts(nrg, m, d, c->z_block_cols > 0 ? c->z_block_cols : d) : 0;
  if (ngp > 0) {                                  // Z and its Gram (the CholQR's) in one launch
    double* Gp = (double*)scratch(c, S_ZGRAM, (size_t)ngp * m * m * sizeof(double));
    double* G = (double*)scratch(c, S_GRAM, (size_t)m * m * sizeof(double));
    if (!Gp || !G) return set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(ngp * ZG_CL));
    cfg.blockDim = dim3(256);
    cfg.stream = c->stream;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = ZG_CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = g_pdl ? 2 : 1;
    const cudaError_t le = cudaLaunchKernelEx(&cfg, reduce_zp_gram_kernel, (const float*)Zp, nrg, dpad, mp, m, d, Z, Gp);
    if (le != cudaSuccess) return check_cuda(c, le, "reduce_zp_gram");
    PPCA_LAUNCH_CHECK(c, "reduce_zp_gram");
    PPCA_TRY(launch_reduce_splits_f64(c, Gp, ngp, (int64_t)m * m, G, c->stream));
    c->zgram_done = true;
    return PPCA_OK;
  }
  launch_reduce_zp(c, Zp, nrg, dpad, mp, m, d, Z);
  PPCA_LAUNCH_CHECK(c, "reduce_zp");
  return PPCA_OK;
}

ppca_status pass_reduce_deferred_s(Ctx* c, double* S, cudaStream_t st) {
  if (!c->s_pending) return PPCA_OK;
  cudaStreamWaitEvent(st, c->s_ev_pass, 0);
  launch_pdl(reduce_spart2_kernel, dim3((unsigned)ceil_div(c->s_m * c->s_m, 32)), dim3(256), 0, st, c->s_part, c->s_parts, c->s_mp,
                                                                               c->s_m, S);
  PPCA_LAUNCH_CHECK(c, "reduce_spart");
  cudaEventRecord(c->s_ev_red, st);
  c->s_pending = false;
  return PPCA_OK;
}

ppca_status pass_tc_power(Ctx* c, const ppca_matrix* X, const PassPlan* plan, const float* W, int m, float* Z, double* S,
                          bool precise) {
  const int mp = pad16(m);
  const int64_t n = X->n_local, d = X->d;
  __nv_bfloat16* Wb;
  float* Wr;
  // reading R30: product 2 of a power pass reads X_hi alone, an error that averages down over the rows
  // (2.9e-5 on the Ritz values at n = 10^5 against the 1e-4 bar, ~1e-4 at n = 2000); below kPreciseRows global
  // rows of a split X the pass adds X_lo·Y_hi (kernel B's XLO instantiation) — the cost is nil at that size
  constexpr int64_t kPreciseRows = 32768;
  precise = precise || (X->dtype == PPCA_F32_SPLIT && X->n_global < kPreciseRows);
  const bool pair = pair_eligible(c, X, mp, precise);
  const bool fused = !pair && fused_eligible(c, X, mp, precise);
  // bf16 X outside the fused kernels and outside the minibatch steps: product 2 with Y_hi alone (R27)
  const bool lean = X->dtype == PPCA_BF16 && !fused && !pair && !precise;
  PPCA_TRY(prep_w(c, W, m, mp, d, &Wb, &Wr));
  const_cast<PassPlan*>(plan)->Wop = Wr;
  if (c->prep_ev) cudaEventRecord(c->prep_ev, c->stream);     // W' ready: the side stream may read Wr
  if (pair) {
    c->last_power_kernel = 4;
    return pass_pair_power(c, X, Wb, m, Z, S);
  }
  if (fused) {
    bool launched = false;
    PPCA_TRY(pass_fused_power(c, X, Wb, m, Z, S, &launched));
    if (launched) {
      c->last_power_kernel = 3;
      return PPCA_OK;
    }
  }
  c->last_power_kernel = 2;
  // Yᵀ as a bf16 pair [Y_hi; Y_lo], [2·mp][ldyt]; kernel A writes every row and column < ldyt
  const int64_t ldyt = ceil_div(n, 64) * 64;
  __nv_bfloat16* YT = (__nv_bfloat16*)scratch(c, S_Y, (size_t)2 * mp * ldyt * 2);
  if (!YT) return set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
  const int64_t nk = ceil_div(d, ka::BK);
  const int ksplit = pick_ksplit(c, X, nk);
  if (ksplit == 1) {
    PPCA_TRY(run_ka(c, X, Wb, m, mp, S, YT, ldyt));
  } else {
    float* Ypart = (float*)scratch(c, S_TC3, (size_t)ksplit * n * mp * sizeof(float));
    if (!Ypart) return set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
    PPCA_TRY(run_ka(c, X, Wb, m, mp, S, nullptr, 0, ksplit, Ypart));
    const int64_t nb = ceil_div(ldyt, (int64_t)YS_RB);
    double* Sp = (double*)scratch(c, S_NTSTAGE, (size_t)nb * m * m * sizeof(double));
    if (!Sp) return set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
    static uint64_t ys_attr = 0;                     // mp = 128: 66 KB of dynamic shared memory
    if (first_on_device(&ys_attr, c->device))
      cudaFuncSetAttribute(ysum_s_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ysum_s_smem(PPCA_MAX_M));
    launch_pdl(ysum_s_kernel, dim3((unsigned)nb), dim3(256), ysum_s_smem(mp), c->stream, Ypart, ksplit, n, mp, m,
                                                                                              YT, ldyt, Sp);
    PPCA_LAUNCH_CHECK(c, "ysum_s");
    PPCA_TRY(launch_reduce_splits_f64(c, Sp, (int)nb, (int64_t)m * m, S));
  }
  // kernel B
  const int nc = kb::Cfg<64>::NC;
  KBParams bp;
  bp.X = X->data; bp.n = n; bp.d = d; bp.ld = X->ld; bp.m = m; bp.mp = mp;
  bp.ndg = ceil_div(d, nc * 128);
  const int64_t ctas = persistent_ctas(c);
  // one work item (d-group × row group) per CTA: the Zᵀ partial stays in TMEM over ~n/(ctas/ndg) rows, so
  // the partials kernel B writes (and reduce_zp reads) are ≈ (ctas/ndg)·d·mp floats
  // (with more d-groups than CTAs, ≥ 4 items per CTA keep the tail short)
  int64_t want = std::max<int64_t>(1, ctas / bp.ndg);
  if (bp.ndg > ctas) {                 // ≥ 4 items per CTA; pick the row-group count with the least tail
    double best = 1e30;
    for (int64_t r = ceil_div(4 * ctas, bp.ndg); r <= ceil_div(4 * ctas, bp.ndg) + 4; ++r) {
      const double items = (double)(bp.ndg * r);
      const double loss = (double)ceil_div(bp.ndg * r, ctas) / (items / (double)ctas);
      if (loss < best - 1e-9) { best = loss; want = r; }
    }
  }
  int64_t rpg = ceil_div(ceil_div(n, want), kb::KR) * kb::KR;
  rpg = std::max<int64_t>(rpg, kb::KR);
  bp.rows_per_rg = rpg;
  bp.nrg = ceil_div(n, rpg);
  const int64_t dpad = bp.ndg * nc * 128;
  float* Zp = (float*)scratch(c, S_PART, (size_t)bp.nrg * dpad * mp * sizeof(float));
  if (!Zp) return set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
  bp.Zp = Zp;
  CUtensorMap tmYT, tmX, tmXlo;
  const int yrows = lean ? mp : 2 * mp;
  if (!make_map_bf16(&tmYT, YT, ldyt, yrows, ldyt, yrows)) return set_error(c, PPCA_ERR_CUDA, "tensor map YT failed");
  tmX = tmYT;
  // product 2 reads X_hi only: bf16 X, or the hi plane of a split X, by TMA
  if (X->dtype != PPCA_F32 && !make_x_maps(X, kb::KR, &tmX, &tmXlo)) return set_error(c, PPCA_ERR_CUDA, "tensor map X failed");
  const int grid = (int)std::min<int64_t>(ctas, bp.ndg * bp.nrg);
  kernel_timer_mark(c, 1);
  if (X->dtype == PPCA_F32)
    PPCA_TRY((dispatch_kb<false, false>(c, mp, tmYT, tmX, tmXlo, bp, grid)));
  else if (precise && X->dtype == PPCA_F32_SPLIT)
    PPCA_TRY((dispatch_kb<true, true>(c, mp, tmYT, tmX, tmXlo, bp, grid)));
  else if (lean)
    PPCA_TRY((dispatch_kb<true, false, true>(c, mp, tmYT, tmX, tmXlo, bp, grid)));
  else
    PPCA_TRY((dispatch_kb<true, false>(c, mp, tmYT, tmX, tmXlo, bp, grid)));
  kernel_timer_mark(c, 1);
  if (c->zp_defer && bp.nrg <= 16 && c->z_block_cols == 0) {   // the EigenGame update sums the partials itself
    c->zp_pending = true;
    c->zp_part = Zp;
    c->zp_nrg = bp.nrg;
    c->zp_dpad = dpad;
    c->zp_mp = mp;
    c->zp_m = m;
    c->zp_d = d;
    return PPCA_OK;
  }
  launch_reduce_zp(c, Zp, bp.nrg, dpad, mp, m, d, Z);
  PPCA_LAUNCH_CHECK(c, "reduce_zp");
  return PPCA_OK;
}

ppca_status pass_reduce_deferred_z(Ctx* c, float* Z) {
  if (!c->zp_pending) return PPCA_OK;
  c->zp_pending = false;
  launch_reduce_zp(c, c->zp_part, c->zp_nrg, c->zp_dpad, c->zp_mp, c->zp_m, c->zp_d, Z);
  PPCA_LAUNCH_CHECK(c, "reduce_zp");
  return PPCA_OK;
}

void pass_tc_release(Ctx*) {}

ppca_status ritz_debug_clocks(unsigned long long* out8);
ppca_status debug_wait_counters(unsigned long long* out16) {
  for (int i = 0; i < 16; ++i) out16[i] = 0;
  return ritz_debug_clocks(out16);             // [0..7]: phase timestamps of the last Ritz-values kernel
}

}  // namespace ppca
