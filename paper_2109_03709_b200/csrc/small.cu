// small.cu — m×m side of the hot path (see small.cuh).  All m×m arithmetic is fp64.
#include <cooperative_groups.h>

#include "small.cuh"
#include "gemm_simt.cuh"

namespace ppca {

// ============================================================================ vector Gram
// G_ij = Σ_x V[i][x] V[j][x] (fp64), the CholQR / operand Gram of the m×m chain (d·m² MAC).
// fp64 FMA throughput bound (64 DFMA / clk / SM): each CTA takes a d-slab, stages GK columns of all m rows
// as fp64 in shared memory ([column][row], so a thread's 8 row values are two 16-byte loads), and every thread
// accumulates one 8×8 register tile of the upper triangle (8 + 8 operand loads per 64 DFMA, warp-broadcast).
// The next stage's fp32 values are loaded into registers while the current one is consumed.  Partials hold
// both triangles of the slab's Gram; launch_reduce_splits_f64 sums the slabs in a fixed order.
constexpr int GK = 32;                            // columns per stage
constexpr int GRAM_MAXT = 160;                    // threads for m ≤ 128: 136 upper 8×8 tiles

template <int MB>                                 // MB = ceil(m / 8) (≤ 16)
__global__ void __launch_bounds__(GRAM_MAXT) vec_gram_tiled_kernel(const float* __restrict__ V, int m, int64_t d,
                                                                   int64_t cols_per_split, double* __restrict__ P) {
  pdl_enter();
  constexpr int MP = MB * 8, LD = MP + 2;         // +2 doubles: 16-byte aligned rows, 4-way worst transposed store
  constexpr int NT = MB * (MB + 1) / 2;           // upper tiles
  constexpr int PER = (MP * GK + GRAM_MAXT - 1) / GRAM_MAXT;
  __shared__ __align__(16) double sv[GK * LD];
  const int64_t xb = (int64_t)blockIdx.x * cols_per_split;
  const int64_t xe = min(d, xb + cols_per_split);
  // tile (bi ≤ bj) of this thread
  int bi = 0, bj = 0;
  {
    int t = threadIdx.x, row = 0;
    while (row < MB && t >= MB - row) { t -= MB - row; ++row; }
    bi = row;
    bj = row + t;
  }
  const bool active = threadIdx.x < NT;
  double acc[8][8];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 8; ++b) acc[a][b] = 0.0;
  float nxt[PER];
  auto fetch = [&](int64_t x0) {
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int e = threadIdx.x + GRAM_MAXT * u;  // e = row·GK + column: a warp reads 32 consecutive columns
      const int r = e / GK, cc = e % GK;
      const int64_t x = x0 + cc;
      nxt[u] = (e < MP * GK && r < m && x < xe) ? __ldg(V + (int64_t)r * d + x) : 0.f;
    }
  };
  if (xb < xe) fetch(xb);
  for (int64_t x0 = xb; x0 < xe; x0 += GK) {
    __syncthreads();                               // the previous stage is consumed
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int e = threadIdx.x + GRAM_MAXT * u;
      if (e < MP * GK) sv[(e % GK) * LD + e / GK] = (double)nxt[u];
    }
    __syncthreads();
    if (x0 + GK < xe) fetch(x0 + GK);              // in flight while this stage is consumed
    if (active) {
#pragma unroll 4
      for (int k = 0; k < GK; ++k) {
        const double2* pa = reinterpret_cast<const double2*>(sv + k * LD + bi * 8);
        const double2* pb = reinterpret_cast<const double2*>(sv + k * LD + bj * 8);
        double a[8], b[8];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double2 va = pa[q], vb = pb[q];
          a[2 * q] = va.x; a[2 * q + 1] = va.y;
          b[2 * q] = vb.x; b[2 * q + 1] = vb.y;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
      }
    }
  }
  if (!active) return;
  double* Pz = P + (int64_t)blockIdx.x * m * m;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int gi = bi * 8 + i, gj = bj * 8 + j;
      if (gi < m && gj < m) {
        Pz[(int64_t)gi * m + gj] = acc[i][j];
        Pz[(int64_t)gj * m + gi] = acc[i][j];      // both triangles (diagonal tiles write the same values twice)
      }
    }
}

// generic 32×32-tile Gram (m > 128: the Prop. 3 checker's stacked [B; T] Gram)
// G_ij = Σ_x V[i][x] V[j][x]; tile 32×32 outputs × 64-column chunks, split over d.
__global__ void __launch_bounds__(256) vec_gram_generic_kernel(const float* __restrict__ V, int m, int64_t d,
                                                       int64_t cols_per_split, double* __restrict__ P) {
  pdl_enter();
  __shared__ double Vi[32][65];                      // staged as fp64: one conversion per staged value, not five
  __shared__ double Vj[32][65];                      // per four DFMAs in the product loop (conversions issue at 1/4 rate)
  const int i0 = blockIdx.x * 32, j0 = blockIdx.y * 32;
  const int64_t xb = (int64_t)blockIdx.z * cols_per_split;
  const int64_t xe = min(d, xb + cols_per_split);
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // ty 0..7 → rows ty*4..+4
  double acc[4] = {0, 0, 0, 0};
  for (int64_t x0 = xb; x0 < xe; x0 += 64) {
    {                                                // 16 loads per thread in flight (clamped, then masked)
      float vi[8], vj[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = threadIdx.x + 256 * u, r = e / 64;
        const int64_t x = min(x0 + e % 64, xe - 1);
        vi[u] = V[(int64_t)min(i0 + r, m - 1) * d + x];
        vj[u] = V[(int64_t)min(j0 + r, m - 1) * d + x];
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = threadIdx.x + 256 * u, r = e / 64, cidx = e % 64;
        const bool xin = x0 + cidx < xe;
        Vi[r][cidx] = (i0 + r < m && xin) ? (double)vi[u] : 0.0;
        Vj[r][cidx] = (j0 + r < m && xin) ? (double)vj[u] : 0.0;
      }
    }
    __syncthreads();
#pragma unroll 8
    for (int cidx = 0; cidx < 64; ++cidx) {
      const double b = Vj[tx][cidx];
#pragma unroll
      for (int a = 0; a < 4; ++a) acc[a] = fma(Vi[ty * 4 + a][cidx], b, acc[a]);
    }
    __syncthreads();
  }
  double* Pz = P + (int64_t)blockIdx.z * m * m;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    int i = i0 + ty * 4 + a, j = j0 + tx;
    if (i < m && j < m) Pz[(int64_t)i * m + j] = acc[a];
  }
}

// m in (120, 128] (C5): the 136 upper 8×8 tiles balanced over 4 warps — one per SM sub-partition, equal work:
// 128 main tiles (the 120 off-diagonal ones and 8 diagonal ones) plus the other 8 diagonal tiles cut into 128
// 2×2 sub-tiles, one per thread (64 + 4 accumulators; the 5-warp kernel above gave one sub-partition two warps).
__global__ void __launch_bounds__(128) vec_gram_bal16_kernel(const float* __restrict__ V, int m, int64_t d,
                                                             int64_t cols_per_split, double* __restrict__ P) {
  pdl_enter();
  constexpr int MP = 128, LD = MP + 2, PER = MP * GK / 128;
  __shared__ __align__(16) double sv[GK * LD];
  const int64_t xb = (int64_t)blockIdx.x * cols_per_split;
  const int64_t xe = min(d, xb + cols_per_split);
  const int t = threadIdx.x;
  int bi, bj;                                      // main tile
  if (t < 120) {                                   // off-diagonal (bi < bj) in row order
    int r = 0, u = t;
    while (u >= 15 - r) { u -= 15 - r; ++r; }
    bi = r;
    bj = r + 1 + u;
  } else {
    bi = bj = t - 120;                             // diagonal tiles 0..7
  }
  // The 8 threads of a quarter warp mostly hold one bi and 8 consecutive bj: their 16-byte loads of tile bj's
  // columns are 64 bytes apart — two bank groups for 8 threads, a 4-way conflict on every b load (ncu: shared
  // wavefronts 69 % of peak, fp64 pipe 28 %).  Thread bj starts its four loads at column pair bj/2 (mod 4), so even
  // and odd bj each cover the four pairs: conflict-free; the accumulator columns are permuted the same way and
  // un-permuted at the store.
  const int rot = (bj >> 1) & 3;
  const int xt = 8 + (t >> 4), xs = t & 15;        // extra: diagonal tile 8..15, 2×2 sub-tile xs
  const int xr = xt * 8 + 2 * (xs >> 2), xc = xt * 8 + 2 * (xs & 3);
  double acc[8][8], ex[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 8; ++b) acc[a][b] = 0.0;
  float nxt[PER];
  auto fetch = [&](int64_t x0) {
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int e = t + 128 * u;
      const int r = e / GK, cc = e % GK;
      const int64_t x = x0 + cc;
      nxt[u] = (r < m && x < xe) ? __ldg(V + (int64_t)r * d + x) : 0.f;
    }
  };
  if (xb < xe) fetch(xb);
  for (int64_t x0 = xb; x0 < xe; x0 += GK) {
    __syncthreads();
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int e = t + 128 * u;
      sv[(e % GK) * LD + e / GK] = (double)nxt[u];
    }
    __syncthreads();
    if (x0 + GK < xe) fetch(x0 + GK);
#pragma unroll 2
    for (int k = 0; k < GK; ++k) {
      const double* row = sv + k * LD;
      const double2* pa = reinterpret_cast<const double2*>(row + bi * 8);
      const double2* pb = reinterpret_cast<const double2*>(row + bj * 8);
      double a[8], b[8];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double2 va = pa[q], vb = pb[(q + rot) & 3];   // b[2q], b[2q+1] = columns 2·((q+rot)&3), +1 of tile bj
        a[2 * q] = va.x; a[2 * q + 1] = va.y;
        b[2 * q] = vb.x; b[2 * q + 1] = vb.y;
      }
      const double2 ea = *reinterpret_cast<const double2*>(row + xr);
      const double2 eb = *reinterpret_cast<const double2*>(row + xc);
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
      ex[0][0] = fma(ea.x, eb.x, ex[0][0]);
      ex[0][1] = fma(ea.x, eb.y, ex[0][1]);
      ex[1][0] = fma(ea.y, eb.x, ex[1][0]);
      ex[1][1] = fma(ea.y, eb.y, ex[1][1]);
    }
  }
  double* Pz = P + (int64_t)blockIdx.x * m * m;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int gi = bi * 8 + i, gj = bj * 8 + 2 * (((j >> 1) + rot) & 3) + (j & 1);
      if (gi < m && gj < m) {
        Pz[(int64_t)gi * m + gj] = acc[i][j];
        Pz[(int64_t)gj * m + gi] = acc[i][j];
      }
    }
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
      if (xr + i < m && xc + j < m) Pz[(int64_t)(xr + i) * m + xc + j] = ex[i][j];   // full diagonal tile
}

// short d (fewer GK-column stages than SMs, e.g. C3's 32) or m > 128: the 32×32-tile kernel over
// (tile, tile, split) keeps more CTAs busy (7.4 vs 9.3 µs at d = 1024, m = 64); otherwise the 8×8-register-tile
// kernel over one d-slab per SM
// (and m ≤ 64: the 8×8-tile kernel would leave most of its threads without a tile — 1 of 160 at m = 8)
static bool gram_short(const Ctx* c, int m, int64_t d) {
  return m > 128 || m <= 64 || ceil_div(d, (int64_t)GK) < c->sm_count;
}

static void vec_gram_split(const Ctx* c, int m, int64_t d, int* nsplit_out, int64_t* cps_out) {
  int64_t cps;
  if (gram_short(c, m, d)) {
    const int tiles = (int)ceil_div(m, 32);
    const int64_t want = ceil_div(2 * (int64_t)c->sm_count, (int64_t)tiles * tiles);
    const int64_t ns = std::max<int64_t>(1, std::min(want, ceil_div(d, (int64_t)64)));
    cps = ceil_div(ceil_div(d, ns), (int64_t)64) * 64;
  } else {
    // m > 120 (vec_gram_bal16_kernel: 128 threads, 255 registers, 34 KB): two slabs per SM, so that two CTAs are
    // co-resident and every sub-partition has two warps to issue DFMAs from (one warp leaves the fp64 pipe idle
    // between its loads)
    static const int per_sm16 = tune_env("PPCA_GRAM_CPSM", 2);
    const int64_t stages = ceil_div(d, (int64_t)GK);
    const int64_t slabs = (int64_t)c->sm_count * (ceil_div(m, 8) >= 16 ? per_sm16 : 1);
    cps = ceil_div(stages, std::min<int64_t>(stages, slabs)) * GK;
  }
  *nsplit_out = (int)ceil_div(d, cps);
  *cps_out = cps;
}

size_t vec_gram_part_bytes(const Ctx* c, int m, int64_t d) {
  int ns;
  int64_t cps;
  vec_gram_split(c, m, d, &ns, &cps);
  return (size_t)ns * m * m * sizeof(double);
}

template <int MB>
static void launch_gram_mb(int nsplit, cudaStream_t st, const float* V, int m, int64_t d, int64_t cps, double* P) {
  launch_pdl(vec_gram_tiled_kernel<MB>, dim3(nsplit), dim3(GRAM_MAXT), 0, st, V, m, d, cps, P);
}

ppca_status vec_gram_on(Ctx* c, const float* V, int m, int64_t d, double* G, cudaStream_t st, int part_slot) {
  int nsplit;
  int64_t cps;
  vec_gram_split(c, m, d, &nsplit, &cps);
  double* P = (double*)scratch(c, part_slot, (size_t)nsplit * m * m * sizeof(double));
  if (!P) return set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
  const int mb = (int)ceil_div(m, 8);
  if (gram_short(c, m, d)) {
    const int tiles = (int)ceil_div(m, 32);
    launch_pdl(vec_gram_generic_kernel, dim3(dim3(tiles, tiles, nsplit)), dim3(256), 0, st, V, m, d, cps, P);
  } else if (mb <= 1) launch_gram_mb<1>(nsplit, st, V, m, d, cps, P);
  else if (mb <= 2) launch_gram_mb<2>(nsplit, st, V, m, d, cps, P);
  else if (mb <= 4) launch_gram_mb<4>(nsplit, st, V, m, d, cps, P);
  else if (mb <= 6) launch_gram_mb<6>(nsplit, st, V, m, d, cps, P);
  else if (mb <= 8) launch_gram_mb<8>(nsplit, st, V, m, d, cps, P);
  else if (mb <= 12) launch_gram_mb<12>(nsplit, st, V, m, d, cps, P);
  else if (mb <= 15) launch_gram_mb<16>(nsplit, st, V, m, d, cps, P);
  else launch_pdl(vec_gram_bal16_kernel, dim3(nsplit), dim3(128), 0, st, V, m, d, cps, P);
  PPCA_LAUNCH_CHECK(c, "vec_gram");
  return launch_reduce_splits_f64(c, P, nsplit, (int64_t)m * m, G, st);
}

ppca_status vec_gram(Ctx* c, const float* V, int m, int64_t d, double* G) {
  return vec_gram_on(c, V, m, d, G, c->stream, S_PART);
}

// ============================================================================ Cholesky (one CTA)
// In smem A[m][lda] (fp64).  Right-looking; pivots ≤ drop²·G_jj are dropped (column zeroed) if
// drop > 0, else flag COLLAPSE.  Writes Linv (lower, dropped rows zero) and keep[] flags.
// (Measured on B200, m = 64, 256 threads: this blocked form 29 µs + 14 µs for L⁻¹; a one-barrier-per-column
// form 45 + 36 µs — its per-step index arithmetic, not the barrier (65 cycles) or rsqrt (62), dominates;
// tools/microbench_small.cu.)
// Blocked right-looking Cholesky in shared memory A[m][m] (fp64, lower, in place), column blocks of CB:
// (1) the diagonal block by one warp (__syncwarp only), (2) the panel below by forward substitution, one
// thread per row, (3) the trailing lower triangle from a transposed copy of the panel (conflict-free).
// Pivots ≤ drop²·G_jj are dropped (column zeroed, keep[j] = 0) when drop > 0, else flag COLLAPSE.
// About 3·m/CB block barriers instead of 2·m column barriers.
constexpr int CB = 16;
__device__ void block_cholesky(double* A, int m, double drop, int* keep, double* diag0, int* d_err, int lda) {
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  __shared__ double rdiag[PPCA_MAX_M];
  __shared__ double panelT[CB][PPCA_MAX_M];
  for (int i = tid; i < m; i += nt) diag0[i] = A[i * lda + i];
  __syncthreads();
  for (int kb = 0; kb < m; kb += CB) {
    const int nb = min(CB, m - kb), ke = kb + nb;
    if (warp == 0) {                              // (1) diagonal block
      for (int j = kb; j < ke; ++j) {
        const double p = A[j * lda + j];
        const bool dr = drop > 0.0 ? !(p > drop * drop * diag0[j]) : (!(p > 0.0) || !isfinite(p));
        // 1/L_jj by one fp64 rsqrt (62 cycles, vs sqrt + divide ≈ 300 on this serial chain), L_jj = p/√p
        const double rp = dr ? 0.0 : rsqrt(p), piv = p * rp;
        const int i = j + 1 + lane;
        const double lij = i < ke ? A[i * lda + j] * rp : 0.0;
        __syncwarp();
        if (lane == 0) {
          A[j * lda + j] = piv;
          keep[j] = !dr;
          rdiag[j] = rp;
          if (dr && drop <= 0.0) atomicOr(d_err, DEV_COLLAPSE);
        }
        if (i < ke) A[i * lda + j] = lij;
        __syncwarp();
        // trailing part of the diagonal block, all lanes at once: lane ↔ (row j+1+(lane&15), columns
        // j+1+(lane>>4)+2t), t < 8; l_kk by shuffle (independent updates, no serial chain)
        {
          const int ir = lane & 15, ii = j + 1 + ir;
          const double li = __shfl_sync(0xffffffffu, lij, ir);
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            const int co = (lane >> 4) + 2 * t, kk = j + 1 + co;
            const double lk = __shfl_sync(0xffffffffu, lij, co & 31);
            if (ii < ke && kk <= ii) A[ii * lda + kk] -= li * lk;
          }
        }
        __syncwarp();
      }
    }
    __syncthreads();
    for (int i = ke + tid; i < m; i += nt) {     // (2) panel rows: L11 x = a_i
      double x[CB];
#pragma unroll
      for (int c = 0; c < CB; ++c) {
        double sum = 0.0;
        if (c < nb) {
          sum = A[i * lda + kb + c];
#pragma unroll
          for (int l = 0; l < c; ++l) sum -= x[l] * A[(kb + c) * lda + kb + l];
          sum *= rdiag[kb + c];
          A[i * lda + kb + c] = sum;
          panelT[c][i] = sum;
        }
        x[c] = sum;
      }
    }
    __syncthreads();
    {                                             // (3) trailing lower triangle
      const int ty = tid >> 4, tx = tid & 15, sy = nt >> 4;
      for (int i = ke + ty; i < m; i += sy) {
        double li[CB];
#pragma unroll
        for (int c = 0; c < CB; ++c) li[c] = c < nb ? A[i * lda + kb + c] : 0.0;
        for (int k = ke + tx; k <= i; k += 16) {
          double acc = 0.0;
#pragma unroll
          for (int c = 0; c < CB; ++c) acc = fma(li[c], c < nb ? panelT[c][k] : 0.0, acc);
          A[i * lda + k] -= acc;
        }
      }
    }
    __syncthreads();
  }
}

// Linv = L⁻¹ (rows of dropped pivots zero) by row blocks of CB: T = Σ_{k < r0} L[r][k]·Linv[k][c] for the
// block's rows and earlier columns (all threads), then a CB-row forward substitution per column (one thread
// per column) with the block's diagonal reciprocals.  2 barriers per row block.
__device__ void block_lower_inverse(const double* L, int m, const int* keep, double* Linv, int lda, int ldi) {
  __shared__ double rd[PPCA_MAX_M];
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int i = tid; i < m; i += nt) rd[i] = (keep[i] && L[i * lda + i] != 0.0) ? 1.0 / L[i * lda + i] : 0.0;
  __syncthreads();
  for (int r0 = 0; r0 < m; r0 += CB) {
    const int nb = min(CB, m - r0);
    for (int e = tid; e < nb * r0; e += nt) {    // T into Linv[r][c], c < r0
      const int r = r0 + e / r0, c = e % r0;
      double a0 = 0.0, a1 = 0.0;
      int k = c;
      for (; k + 1 < r0; k += 2) {
        a0 = fma(L[r * lda + k], Linv[(int64_t)k * ldi + c], a0);
        a1 = fma(L[r * lda + k + 1], Linv[(int64_t)(k + 1) * ldi + c], a1);
      }
      if (k < r0) a0 = fma(L[r * lda + k], Linv[(int64_t)k * ldi + c], a0);
      Linv[(int64_t)r * ldi + c] = a0 + a1;
    }
    __syncthreads();
    for (int c = tid; c < m; c += nt) {           // forward substitution within the row block
      double x[CB];
#pragma unroll
      for (int rr = 0; rr < CB; ++rr) {
        double v = 0.0;
        if (rr < nb) {
          const int r = r0 + rr;
          if (c <= r) {
            double rhs = c < r0 ? -Linv[(int64_t)r * ldi + c] : (r == c ? 1.0 : 0.0);
#pragma unroll
            for (int l = 0; l < rr; ++l) rhs -= L[r * lda + r0 + l] * x[l];
            v = rhs * rd[r];
          }
          Linv[(int64_t)r * ldi + c] = v;
        }
        x[rr] = v;
      }
    }
    __syncthreads();
  }
}

__device__ unsigned long long g_chol_clk[8];     // phase clocks of the last chol_inv (profiling)

__global__ void chol_inv_kernel(const double* __restrict__ G, int m, double drop, double* __restrict__ Linv,
                                int* __restrict__ row_map, int* __restrict__ m_out, int* d_err) {
  pdl_enter();
  extern __shared__ double sm[];
  if (threadIdx.x == 0) g_chol_clk[0] = clock64();
  const int lda = m | 1;                           // odd row stride: column walks hit distinct banks
  double* A = sm;                                  // m × lda
  double* diag0 = A + m * lda;                     // m
  int* keep = (int*)(diag0 + m);                   // m
  double* Ls = reinterpret_cast<double*>(keep + ((m + 1) & ~1));   // m × lda when m ≤ 90 (L⁻¹ built in smem)
  const bool in_smem = m <= 90;
  copy_batched<16>(threadIdx.x, m * m, blockDim.x, [&](int64_t e) { return G[e]; },
                   [&](int64_t e, double v) { A[(e / m) * lda + e % m] = v; });
  __syncthreads();
  if (threadIdx.x == 0) g_chol_clk[1] = clock64();
  block_cholesky(A, m, drop, keep, diag0, d_err, lda);
  if (threadIdx.x == 0) g_chol_clk[2] = clock64();
  if (in_smem) {
    block_lower_inverse(A, m, keep, Ls, lda, lda);
    if (threadIdx.x == 0) g_chol_clk[3] = clock64();
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) Linv[e] = Ls[(e / m) * lda + e % m];
  } else {
    block_lower_inverse(A, m, keep, Linv, lda, m);
    if (threadIdx.x == 0) g_chol_clk[3] = clock64();
  }
  if (threadIdx.x == 0) g_chol_clk[4] = clock64();
  if (threadIdx.x == 0) {
    int o = 0;
    for (int i = 0; i < m; ++i) row_map[i] = keep[i] ? o++ : -1;
    *m_out = o;
  }
}

// No-drop Cholesky and L⁻¹ in one register-resident sweep (m ≤ 64; the power step's re-orthonormalisation).
// Right-looking elimination on [A | M], M = I initially: at step j, with p = A_jj,
//   A_ik −= A_ij A_kj / p  (i, k > j),   M_j· ← M_j· / √p,   M_i· −= (A_ij / p) M_j·  (i > j, M_j· unscaled),
// so that M = L⁻¹ at the end (forward substitution of L Y = I, row-oriented).  Thread t owns row t/CQ and the
// columns ≡ t (mod CQ) of both A and M (64/CQ + 64/CQ fp64 registers; CQ = 8, 512 threads: 21 µs in ncu
// against 29 µs for CQ = 4 and 27 µs for CQ = 16); column j of A and row j of M go through
// double-buffered shared memory — one barrier per step, no index arithmetic in the loop (the blocked
// shared-memory version's cost, tools/microbench_small.cu).  Rows/columns ≥ m are the identity.
constexpr int CF_M = 64;
static const bool g_chol_reg = tune_env("PPCA_CHOL_REG", 1) != 0;
// the sweep as a block-level device function (blockDim.x == 64·CQ): G [m][m] and Linv [m][ldl] in any
// memory space; keep[i] = 1 (no drops); a non-positive pivot flags DEV_COLLAPSE.  Used by the CholQR kernel
// below and by the Ritz kernels (ritz.cuh) for the operand Gram's L⁻¹.
template <int CQ>
__device__ void chol_inv_sweep(const double* __restrict__ G, int m, double* __restrict__ Linv, int ldl,
                               int* __restrict__ keep, int* d_err, int ldg = -1) {
  if (ldg < 0) ldg = m;
  __shared__ double colb[2][CF_M];
  __shared__ double rowb[2][CF_M];
  constexpr int NQ = CF_M / CQ;
  const int t = threadIdx.x, i = t / CQ, cp = t % CQ;
  double a[NQ], mm_[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int k = cp + CQ * q;
    a[q] = (i < m && k < m) ? G[i * ldg + k] : (i == k ? 1.0 : 0.0);
    mm_[q] = i == k ? 1.0 : 0.0;
  }
  // step 0's buffers
  if (cp == 0) colb[0][i] = a[0];
  if (i == 0) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) rowb[0][cp + CQ * q] = mm_[q];
  }
  __syncthreads();
  bool bad = false;
  // fully unrolled: every register index is static, and the updates that only touch finished columns of A
  // (k < j) or the zero upper triangle of M (c > j) are dropped at compile time
#pragma unroll
  for (int j = 0; j < CF_M; ++j) {
    const int b = j & 1;
    const double p = colb[b][j];
    const bool ok = p > 0.0 && isfinite(p);
    bad |= !ok;
    const double r = ok ? rsqrt(p) : 0.0;
    // row i > j: M_i −= (A_ij/p)·M_j;  row j: M_j ← r·M_j = M_j − (1 − r)·M_j (rowb holds M_j);  rows < j: 0.
    // colb rows < j are published as zero, so f needs no mask there.
    const double f = i == j ? 1.0 - r : colb[b][i] * (r * r);
    const double fa = i > j ? f : 0.0;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      if (CQ * q + CQ - 1 > j) a[q] = fma(-fa, colb[b][cp + CQ * q], a[q]);
      if (CQ * q <= j) mm_[q] = fma(-f, rowb[b][cp + CQ * q], mm_[q]);
    }
    if (j + 1 < CF_M) {                              // publish column j+1 of A and row j+1 of M
      const int jn = j + 1, nb = b ^ 1;
      if (cp == jn % CQ) colb[nb][i] = i >= jn ? a[jn / CQ] : 0.0;
      if (i == jn) {
#pragma unroll
        for (int q = 0; q < NQ; ++q)
          if (CQ * q <= jn) rowb[nb][cp + CQ * q] = mm_[q];
      }
    }
    __syncthreads();
  }
  if (bad && t == 0) atomicOr(d_err, DEV_COLLAPSE);
  if (i < m) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int k = cp + CQ * q;
      if (k < m) Linv[i * ldl + k] = mm_[q];
    }
  }
  if (keep && t < m) keep[t] = 1;
  __syncthreads();
}

// The same elimination two steps per barrier (steps j and j+1 from columns j, j+1 of A and rows j, j+1 of M as
// they stand before step j): every thread forms column j+1 and row j+1 after step j itself — with the operation
// order of the one-step sweep, so the result is bitwise the same — and applies both updates:
//   p1 = A_{j+1,j+1} − h·A_{j+1,j} (h = A_{j+1,j}/p0),  c1'_i = A_{i,j+1} − (A_ij/p0)·A_{j+1,j},
//   A_ik −= (A_ij/p0)·A_kj + (c1'_i/p1)·c1'_k  (i, k > j+1),
//   M_i· −= F0_i·M_j·, then −= F1_i·(M_{j+1}· − h·M_j·)  (F0_j = 1 − r0, F1_{j+1} = 1 − r1, the rest as above).
// Half the barriers and publications of chol_inv_sweep; the two rsqrt stay sequential.
template <int CQ>
__device__ void chol_inv_sweep2(const double* __restrict__ G, int m, double* __restrict__ Linv, int ldl, int* d_err) {
  static_assert(CQ >= 2, "columns j and j+1 have different owners");
  __shared__ double colb[2][2][CF_M];
  __shared__ double rowb[2][2][CF_M];
  constexpr int NQ = CF_M / CQ;
  const int t = threadIdx.x, i = t / CQ, cp = t % CQ;
  double a[NQ], mm_[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int k = cp + CQ * q;
    a[q] = (i < m && k < m) ? G[i * m + k] : (i == k ? 1.0 : 0.0);
    mm_[q] = i == k ? 1.0 : 0.0;
  }
  if (cp == 0) colb[0][0][i] = a[0];
  if (cp == 1) colb[0][1][i] = a[0];
  if (i < 2) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) rowb[0][i][cp + CQ * q] = mm_[q];
  }
  __syncthreads();
  bool bad = false;
#pragma unroll
  for (int j = 0; j < CF_M; j += 2) {
    const int b = (j >> 1) & 1;
    const double p0 = colb[b][0][j];
    const double c0j1 = colb[b][0][j + 1];
    const double c1j1 = colb[b][1][j + 1];
    const double c0i = colb[b][0][i], c1i = colb[b][1][i];
    const bool ok0 = p0 > 0.0 && isfinite(p0);
    const double r0 = ok0 ? rsqrt(p0) : 0.0;
    const double g0 = r0 * r0;
    const double h = c0j1 * g0;
    const double p1 = fma(-h, c0j1, c1j1);
    const bool ok1 = p1 > 0.0 && isfinite(p1);
    const double r1 = ok1 ? rsqrt(p1) : 0.0;
    const double g1 = r1 * r1;
    bad |= !ok0 || !ok1;
    const double f0 = c0i * g0;
    const double c1pi = fma(-f0, c0j1, c1i);
    const double F0 = i == j ? 1.0 - r0 : f0;
    const double F1 = i == j + 1 ? 1.0 - r1 : (i > j + 1 ? c1pi * g1 : 0.0);
    const bool live = i > j + 1;
    const double fa0 = live ? f0 : 0.0, fa1 = live ? c1pi * g1 : 0.0;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int kk = cp + CQ * q;
      if (CQ * q + CQ - 1 >= j + 2) {             // columns k ≥ j+2 of A
        const double c0k = colb[b][0][kk];
        const double c1k = fma(-(c0k * g0), c0j1, colb[b][1][kk]);
        a[q] = fma(-fa0, c0k, a[q]);
        a[q] = fma(-fa1, c1k, a[q]);
      }
      if (CQ * q <= j + 1) {                      // rows j, j+1 of M have entries k ≤ j+1 only
        const double mj = rowb[b][0][kk];
        const double mj1 = fma(-h, mj, rowb[b][1][kk]);
        mm_[q] = fma(-F0, mj, mm_[q]);
        mm_[q] = fma(-F1, mj1, mm_[q]);
      }
    }
    if (j + 2 < CF_M) {                          // publish columns j+2, j+3 of A and rows j+2, j+3 of M
      const int jn = j + 2, nb = b ^ 1;
      if (cp == jn % CQ) colb[nb][0][i] = i >= jn ? a[jn / CQ] : 0.0;
      if (cp == (jn + 1) % CQ) colb[nb][1][i] = i >= jn ? a[(jn + 1) / CQ] : 0.0;
      if (i == jn || i == jn + 1) {
#pragma unroll
        for (int q = 0; q < NQ; ++q)
          if (CQ * q <= jn + 1) rowb[nb][i - jn][cp + CQ * q] = mm_[q];
      }
    }
    __syncthreads();
  }
  if (bad && t == 0) atomicOr(d_err, DEV_COLLAPSE);
  if (i < m) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int k = cp + CQ * q;
      if (k < m) Linv[i * ldl + k] = mm_[q];
    }
  }
  __syncthreads();
}

// chol_inv_sweep2 with the two published columns (and the two M rows) interleaved as double2: one 16-byte
// shared load gives a thread both operands of a column index (the sweep is bound by its shared-memory loads:
// every thread reads the published column and row at its 2·64/CQ indices each step).  Bitwise the same result.
template <int CQ>
__device__ void chol_inv_sweep2p(const double* __restrict__ G, int m, double* __restrict__ Linv, int ldl, int* d_err) {
  static_assert(CQ >= 2, "columns j and j+1 have different owners");
  __shared__ double2 colb[2][CF_M];
  __shared__ double2 rowb[2][CF_M];
  constexpr int NQ = CF_M / CQ;
  const int t = threadIdx.x, i = t / CQ, cp = t % CQ;
  double a[NQ], mm_[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int k = cp + CQ * q;
    a[q] = (i < m && k < m) ? G[i * m + k] : (i == k ? 1.0 : 0.0);
    mm_[q] = i == k ? 1.0 : 0.0;
  }
  if (cp == 0) colb[0][i].x = a[0];
  if (cp == 1) colb[0][i].y = a[0];
  if (i < 2) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      if (i == 0) rowb[0][cp + CQ * q].x = mm_[q];
      else rowb[0][cp + CQ * q].y = mm_[q];
    }
  }
  __syncthreads();
  bool bad = false;
#pragma unroll
  for (int j = 0; j < CF_M; j += 2) {
    const int b = (j >> 1) & 1;
    const double p0 = colb[b][j].x;
    const double2 cj1 = colb[b][j + 1];
    const double c0j1 = cj1.x, c1j1 = cj1.y;
    const double2 ci = colb[b][i];
    const double c0i = ci.x, c1i = ci.y;
    const bool ok0 = p0 > 0.0 && isfinite(p0);
    const double r0 = ok0 ? rsqrt(p0) : 0.0;
    const double g0 = r0 * r0;
    const double h = c0j1 * g0;
    const double p1 = fma(-h, c0j1, c1j1);
    const bool ok1 = p1 > 0.0 && isfinite(p1);
    const double r1 = ok1 ? rsqrt(p1) : 0.0;
    const double g1 = r1 * r1;
    bad |= !ok0 || !ok1;
    const double f0 = c0i * g0;
    const double c1pi = fma(-f0, c0j1, c1i);
    const double F0 = i == j ? 1.0 - r0 : f0;
    const double F1 = i == j + 1 ? 1.0 - r1 : (i > j + 1 ? c1pi * g1 : 0.0);
    const bool live = i > j + 1;
    const double fa0 = live ? f0 : 0.0, fa1 = live ? c1pi * g1 : 0.0;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int kk = cp + CQ * q;
      if (CQ * q + CQ - 1 >= j + 2) {
        const double2 ck = colb[b][kk];
        const double c1k = fma(-(ck.x * g0), c0j1, ck.y);
        a[q] = fma(-fa0, ck.x, a[q]);
        a[q] = fma(-fa1, c1k, a[q]);
      }
      if (CQ * q <= j + 1) {
        const double2 mk = rowb[b][kk];
        const double mj1 = fma(-h, mk.x, mk.y);
        mm_[q] = fma(-F0, mk.x, mm_[q]);
        mm_[q] = fma(-F1, mj1, mm_[q]);
      }
    }
    if (j + 2 < CF_M) {
      const int jn = j + 2, nb = b ^ 1;
      if (cp == jn % CQ) colb[nb][i].x = i >= jn ? a[jn / CQ] : 0.0;
      if (cp == (jn + 1) % CQ) colb[nb][i].y = i >= jn ? a[(jn + 1) / CQ] : 0.0;
      if (i == jn) {
#pragma unroll
        for (int q = 0; q < NQ; ++q)
          if (CQ * q <= jn + 1) rowb[nb][cp + CQ * q].x = mm_[q];
      } else if (i == jn + 1) {
#pragma unroll
        for (int q = 0; q < NQ; ++q)
          if (CQ * q <= jn + 1) rowb[nb][cp + CQ * q].y = mm_[q];
      }
    }
    __syncthreads();
  }
  if (bad && t == 0) atomicOr(d_err, DEV_COLLAPSE);
  if (i < m) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int k = cp + CQ * q;
      if (k < m) Linv[i * ldl + k] = mm_[q];
    }
  }
  __syncthreads();
}

// The packed two-step sweep on register tiles: thread = RI consecutive rows × the columns ≡ cp (mod CQ) of A and of
// M ((64/RI)·CQ threads; threads beyond that only take part in the barriers).  chol_inv_sweep2p delivers
// 64·64·2·16 B = 128 KB of published operands to registers per step whatever its CQ (every element loads its own
// column's double2: ≈ 1000 cycles of the 128 B/clk shared-memory pipe — the measured 0.9 µs per step); a thread
// that owns RI rows loads each column operand once for all of them: (2·64/CQ + RI + 2) 16-byte loads per thread,
// 56 KB per step for RI = 4, CQ = 16.  Threads whose rows are all finished (< j) skip the step's arithmetic and
// loads.  Every element sees the operations of chol_inv_sweep2p in the same order: bitwise the same L⁻¹.
template <int RI, int CQ>
__device__ void chol_inv_sweep2t(const double* __restrict__ G, int m, double* __restrict__ Linv, int ldl, int* d_err,
                                 int ldg = -1, int* __restrict__ keep = nullptr) {
  static_assert(CQ >= 2 && RI >= 2 && RI % 2 == 0 && CF_M % RI == 0 && CF_M % CQ == 0, "tile shape");
  if (ldg < 0) ldg = m;
  __shared__ double2 colb[2][CF_M];
  __shared__ double2 rowb[2][CF_M];
  constexpr int NQ = CF_M / CQ;
  constexpr int NT = (CF_M / RI) * CQ;
  const int t = threadIdx.x, ig = t / CQ, cp = t % CQ, i0 = ig * RI;
  const bool act = t < NT;
  double a[RI][NQ], mm_[RI][NQ];
  if (act) {
#pragma unroll
    for (int r = 0; r < RI; ++r)
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const int i = i0 + r, k = cp + CQ * q;
        a[r][q] = (i < m && k < m) ? G[i * ldg + k] : (i == k ? 1.0 : 0.0);
        mm_[r][q] = i == k ? 1.0 : 0.0;
      }
    if (cp == 0) {
#pragma unroll
      for (int r = 0; r < RI; ++r) colb[0][i0 + r].x = a[r][0];
    }
    if (cp == 1) {
#pragma unroll
      for (int r = 0; r < RI; ++r) colb[0][i0 + r].y = a[r][0];
    }
    if (ig == 0) {
#pragma unroll
      for (int q = 0; q < NQ; ++q) rowb[0][cp + CQ * q] = make_double2(mm_[0][q], mm_[1][q]);
    }
  }
  __syncthreads();
  bool bad = false;
#pragma unroll
  for (int j = 0; j < CF_M; j += 2) {
    const int b = (j >> 1) & 1;
    if (act && i0 + RI - 1 >= j) {                   // rows < j are finished in A and in M
      const double p0 = colb[b][j].x;
      const double2 cj1 = colb[b][j + 1];
      const double c0j1 = cj1.x, c1j1 = cj1.y;
      const bool ok0 = p0 > 0.0 && isfinite(p0);
      const double r0 = ok0 ? rsqrt(p0) : 0.0;
      const double g0 = r0 * r0;
      const double h = c0j1 * g0;
      const double p1 = fma(-h, c0j1, c1j1);
      const bool ok1 = p1 > 0.0 && isfinite(p1);
      const double r1 = ok1 ? rsqrt(p1) : 0.0;
      const double g1 = r1 * r1;
      bad |= !ok0 || !ok1;
      double F0[RI], F1[RI], fa0[RI], fa1[RI];
#pragma unroll
      for (int r = 0; r < RI; ++r) {
        const int i = i0 + r;
        const double2 ci = colb[b][i];
        const double f0 = ci.x * g0;
        const double c1pi = fma(-f0, c0j1, ci.y);
        const bool live = i > j + 1;
        F0[r] = i == j ? 1.0 - r0 : f0;
        F1[r] = i == j + 1 ? 1.0 - r1 : (live ? c1pi * g1 : 0.0);
        fa0[r] = live ? f0 : 0.0;
        fa1[r] = live ? c1pi * g1 : 0.0;
      }
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const int kk = cp + CQ * q;
        if (CQ * q + CQ - 1 >= j + 2) {
          const double2 ck = colb[b][kk];
          const double c1k = fma(-(ck.x * g0), c0j1, ck.y);
#pragma unroll
          for (int r = 0; r < RI; ++r) {
            a[r][q] = fma(-fa0[r], ck.x, a[r][q]);
            a[r][q] = fma(-fa1[r], c1k, a[r][q]);
          }
        }
        if (CQ * q <= j + 1) {
          const double2 mk = rowb[b][kk];
          const double mj1 = fma(-h, mk.x, mk.y);
#pragma unroll
          for (int r = 0; r < RI; ++r) {
            mm_[r][q] = fma(-F0[r], mk.x, mm_[r][q]);
            mm_[r][q] = fma(-F1[r], mj1, mm_[r][q]);
          }
        }
      }
      if (j + 2 < CF_M) {                            // publish columns j+2, j+3 of A and rows j+2, j+3 of M
        const int jn = j + 2, nb = b ^ 1;
        if (cp == jn % CQ) {
#pragma unroll
          for (int r = 0; r < RI; ++r) colb[nb][i0 + r].x = i0 + r >= jn ? a[r][jn / CQ] : 0.0;
        }
        if (cp == (jn + 1) % CQ) {
#pragma unroll
          for (int r = 0; r < RI; ++r) colb[nb][i0 + r].y = i0 + r >= jn ? a[r][(jn + 1) / CQ] : 0.0;
        }
        if (ig == jn / RI) {
#pragma unroll
          for (int q = 0; q < NQ; ++q)
            if (CQ * q <= jn + 1) rowb[nb][cp + CQ * q] = make_double2(mm_[jn % RI][q], mm_[jn % RI + 1][q]);
        }
      }
    }
    __syncthreads();
  }
  if (__syncthreads_or(bad) && t == 0) atomicOr(d_err, DEV_COLLAPSE);
  if (act) {
#pragma unroll
    for (int r = 0; r < RI; ++r)
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const int i = i0 + r, k = cp + CQ * q;
        if (i < m && k < m) Linv[i * ldl + k] = mm_[r][q];
      }
  }
  if (keep && t < m) keep[t] = 1;
  __syncthreads();
}

template <int RI, int CQ>
__global__ void __launch_bounds__((CF_M / RI) * CQ) chol_inv_regt_kernel(const double* __restrict__ G, int m,
                                                                      double* __restrict__ Linv,
                                                                      int* __restrict__ row_map,
                                                                      int* __restrict__ m_out, int* d_err) {
  pdl_enter();
  chol_inv_sweep2t<RI, CQ>(G, m, Linv, m, d_err);
  for (int i = threadIdx.x; i < m; i += blockDim.x) row_map[i] = i;
  if (threadIdx.x == 0) *m_out = m;
}

// 0 one-step, 1 two-step, 2 two-step packed, 3–6 packed on register tiles of (2, 4), (4, 4), (4, 8), (2, 8) rows ×
// columns per thread.  Same box, C3 chain (profiles/r2_s6_chol_tiles_ab.txt): 2: 35.5 µs, 3: 26.5 µs, 4: 37.5 µs,
// 5: 47 µs, 6: 35 µs from the Gram's split sum to the sweep's end — the sweep needs the 512 threads (latency), and
// two rows per thread take a third off its shared-memory loads
static const int g_chol2 = tune_env("PPCA_CHOL2", 3);

template <int CQ>
__global__ void __launch_bounds__(64 * CQ) chol_inv_reg_kernel(const double* __restrict__ G, int m,
                                                           double* __restrict__ Linv, int* __restrict__ row_map,
                                                           int* __restrict__ m_out, int* d_err, int variant) {
  pdl_enter();
  if (variant == 2) chol_inv_sweep2p<CQ>(G, m, Linv, m, d_err);
  else if (variant == 1) chol_inv_sweep2<CQ>(G, m, Linv, m, d_err);
  else chol_inv_sweep<CQ>(G, m, Linv, m, nullptr, d_err);
  if (threadIdx.x < m) row_map[threadIdx.x] = threadIdx.x;
  if (threadIdx.x == 0) *m_out = m;
}

// 64 < m ≤ 128 (C5's m = 128): 2×2 blocks of 64 around the register sweep, one CTA of 512 threads —
//   L11⁻¹ = sweep(A11);  L21 = A21·L11⁻ᵀ;  A22' = A22 − L21·L21ᵀ;  L22⁻¹ = sweep(A22');
//   L⁻¹ = [[L11⁻¹, 0], [−L22⁻¹·L21·L11⁻¹, L22⁻¹]]
// (four 64³ fp64 products in shared memory between two sweeps; the one-CTA blocked elimination it replaces
// took 153 µs at m = 128).
constexpr int BK64 = 64, BKL = BK64 + 1;
__device__ __forceinline__ void mm64(const double* __restrict__ A, bool at, const double* __restrict__ B, bool bt,
                                     double* __restrict__ C, double alpha, const double* __restrict__ Cin, int ldcin) {
  // C[i][j] = Cin[i][j] + alpha·Σ_k opA[i][k]·opB[k][j]  (64×64, ld BKL; op = transpose when flagged; Cin may be
  // null); 512 threads × 8 outputs, rows i = t/8, columns j = t%8 + 8q
  const int i = threadIdx.x >> 3, j0 = threadIdx.x & 7;
  double acc[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) acc[q] = 0.0;
  for (int k = 0; k < BK64; ++k) {
    const double a = at ? A[k * BKL + i] : A[i * BKL + k];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = fma(a, bt ? B[(j0 + 8 * q) * BKL + k] : B[k * BKL + j0 + 8 * q], acc[q]);
  }
  __syncthreads();                                 // C may alias an operand's storage of an earlier phase
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int j = j0 + 8 * q;
    C[i * BKL + j] = (Cin ? Cin[i * ldcin + j] : 0.0) + alpha * acc[q];
  }
  __syncthreads();
}

__global__ void __launch_bounds__(512) chol_inv_blk_kernel(const double* __restrict__ G, int m, double* __restrict__ Linv,
                                                           int* __restrict__ row_map, int* __restrict__ m_out,
                                                           int* d_err) {
  pdl_enter();
  extern __shared__ double cb[];
  double* L11i = cb;                              // L11⁻¹
  double* L21 = L11i + BK64 * BKL;                  // A21, then L21
  double* A22 = L21 + BK64 * BKL;                   // A22', then T = L21·L11⁻¹
  double* L22i = A22 + BK64 * BKL;                  // L22⁻¹
  const int m2 = m - BK64;
  chol_inv_sweep2t<2, 16>(G, BK64, L11i, BKL, d_err, m);
  for (int e = threadIdx.x; e < BK64 * BK64; e += 512) {            // A21 (rows ≥ m2 zero)
    const int i = e / BK64, k = e % BK64;
    A22[i * BKL + k] = i < m2 ? G[(BK64 + i) * m + k] : 0.0;
  }
  __syncthreads();
  mm64(A22, false, L11i, true, L21, 1.0, nullptr, 0);            // L21 = A21·L11⁻ᵀ
  for (int e = threadIdx.x; e < BK64 * BK64; e += 512) {            // A22 (identity beyond m2)
    const int i = e / BK64, k = e % BK64;
    L22i[i * BKL + k] = (i < m2 && k < m2) ? G[(BK64 + i) * m + BK64 + k] : (i == k ? 1.0 : 0.0);
  }
  __syncthreads();
  mm64(L21, false, L21, true, A22, -1.0, L22i, BKL);             // A22' = A22 − L21·L21ᵀ
  chol_inv_sweep2t<2, 16>(A22, m2, L22i, BKL, d_err, BKL);
  mm64(L21, false, L11i, false, A22, 1.0, nullptr, 0);           // T = L21·L11⁻¹
  mm64(L22i, false, A22, false, L21, -1.0, nullptr, 0);          // X21 = −L22⁻¹·T
  for (int e = threadIdx.x; e < m * m; e += 512) {
    const int i = e / m, k = e % m;
    double v;
    if (i < BK64) v = k < BK64 ? L11i[i * BKL + k] : 0.0;
    else v = k < BK64 ? L21[(i - BK64) * BKL + k] : L22i[(i - BK64) * BKL + (k - BK64)];
    Linv[e] = v;
  }
  if (threadIdx.x < m) row_map[threadIdx.x] = threadIdx.x;
  if (threadIdx.x == 0) *m_out = m;
}

static int g_chol_cq = tune_env("PPCA_CHOL_CQ", 8);
static void launch_chol_inv_reg(const double* G, int m, double* Linv, int* row_map, int* m_out, int* d_err,
                                cudaStream_t st) {
  if (m > CF_M) {
    const size_t smem = (size_t)4 * BK64 * BKL * sizeof(double);
    int dev = 0;
    cudaGetDevice(&dev);
    static uint64_t attr = 0;
    if (first_on_device(&attr, dev))
      cudaFuncSetAttribute(chol_inv_blk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    launch_pdl(chol_inv_blk_kernel, dim3(1), dim3(512), smem, st, G, m, Linv, row_map, m_out, d_err);
    return;
  }
  if (g_chol2 == 3) {        // register tiles: 2 rows × 4 columns, 512 threads
    launch_pdl(chol_inv_regt_kernel<2, 16>, dim3(1), dim3(512), 0, st, G, m, Linv, row_map, m_out, d_err);
    return;
  }
  if (g_chol2 == 4) {        // 4 rows × 4 columns, 256 threads
    launch_pdl(chol_inv_regt_kernel<4, 16>, dim3(1), dim3(256), 0, st, G, m, Linv, row_map, m_out, d_err);
    return;
  }
  if (g_chol2 == 5) {        // 4 rows × 8 columns, 128 threads
    launch_pdl(chol_inv_regt_kernel<4, 8>, dim3(1), dim3(128), 0, st, G, m, Linv, row_map, m_out, d_err);
    return;
  }
  if (g_chol2 == 6) {        // 2 rows × 8 columns, 256 threads
    launch_pdl(chol_inv_regt_kernel<2, 8>, dim3(1), dim3(256), 0, st, G, m, Linv, row_map, m_out, d_err);
    return;
  }
  if (g_chol_cq == 4)
    launch_pdl(chol_inv_reg_kernel<4>, dim3(1), dim3(256), 0, st, G, m, Linv, row_map, m_out, d_err, g_chol2);
  else if (g_chol_cq == 16)
    launch_pdl(chol_inv_reg_kernel<16>, dim3(1), dim3(1024), 0, st, G, m, Linv, row_map, m_out, d_err, g_chol2);
  else
    launch_pdl(chol_inv_reg_kernel<8>, dim3(1), dim3(512), 0, st, G, m, Linv, row_map, m_out, d_err, g_chol2);
}

static size_t chol_inv_smem(int m) {
  const int lda = m | 1;
  return (size_t)m * lda * sizeof(double) + m * sizeof(double) + ((m + 1) & ~1) * sizeof(int) +
         (m <= 90 ? (size_t)m * lda * sizeof(double) : 0);
}

// ============================================================================ apply: OUT = C · IN
// OUT[row_map(i)] = Σ_j C[i][j]·IN[j] for i < rows (C fp64 [rows][ldc], IN [m_in][d] fp32, fp64 accumulation;
// lower: C lower-triangular).  The apply of CholQR (W = L⁻¹Z, d·m²/2 MAC), the lift E = R·B and the EigenGame
// mixing.  fp64-FMA bound: a grid of ≤ one CTA per SM, each holding Cᵀ in shared memory once and sweeping
// 32-column chunks of IN; thread = RPT rows × 4 columns of the output chunk (RPT + 4 operand loads per 4·RPT
// DFMA, warp-broadcast), the next chunk's IN loaded into registers while the current one is consumed.
// short d (fewer 32-column chunks than SMs, e.g. C3's d = 1024): one CTA per 32 columns × row blocks, C
// staged per CTA (measured faster there than the chunk-sweeping kernel below: 8.1 vs 11.6 µs for m = 64)
// element e of the next pass operand W' = [W_hi; W_lo] (lo rows at lo_off) and W_r = hi + lo from the fp32 value
// o, exactly as prep_w_kernel splits it (RN conversions, residual in fp32)
__device__ __forceinline__ void split_store(__nv_bfloat16* Wb, float* Wr, int64_t lo_off, int64_t e, float o) {
  const __nv_bfloat16 h = __float2bfloat16_rn(o);
  const float hf = __bfloat162float(h);
  const __nv_bfloat16 l = __float2bfloat16_rn(o - hf);
  Wb[e] = h;
  Wb[lo_off + e] = l;
  Wr[e] = hf + __bfloat162float(l);
}

constexpr int AP_COLS = 32;
__global__ void __launch_bounds__(256) apply_rows_kernel(const double* __restrict__ C, int ldc, int rows,
                                                         int m_in, const int* __restrict__ row_map,
                                                         bool lower, const float* __restrict__ IN,
                                                         int64_t d, float* __restrict__ OUT, int rows_per_cta,
                                                         __nv_bfloat16* __restrict__ Wb, float* __restrict__ Wr,
                                                         int64_t lo_off) {
  pdl_enter();
  extern __shared__ double cs[];                 // this CTA's rows × m_in (fp64), then m_in × AP_COLS (fp32)
  const int r0 = blockIdx.y * rows_per_cta, r1 = min(rows, r0 + rows_per_cta);
  float* ins = reinterpret_cast<float*>(cs + (size_t)rows_per_cta * m_in);
  const int64_t x0 = (int64_t)blockIdx.x * AP_COLS;
  copy_batched<16>(threadIdx.x, (r1 - r0) * m_in, blockDim.x,
                   [&](int64_t e) { return C[(r0 + e / m_in) * ldc + e % m_in]; },
                   [&](int64_t e, double v) { cs[e] = v; });
  copy_batched<8>(threadIdx.x, m_in * AP_COLS, blockDim.x,
                  [&](int64_t e) {
                    const int64_t x = x0 + e % AP_COLS;
                    return IN[(e / AP_COLS) * d + (x < d ? x : d - 1)];
                  },
                  [&](int64_t e, float v) { ins[e] = x0 + e % AP_COLS < d ? v : 0.f; });
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t x = x0 + lane;
  for (int i = r0 + warp; i < r1; i += 8) {
    const int oi = row_map ? row_map[i] : i;
    if (oi < 0) continue;
    const double* crow = cs + (size_t)(i - r0) * m_in;
    const int jend = lower ? min(i + 1, m_in) : m_in;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;   // four chains: the FMA latency is hidden
    int j = 0;
    for (; j + 4 <= jend; j += 4) {
      a0 = fma(crow[j], (double)ins[j * AP_COLS + lane], a0);
      a1 = fma(crow[j + 1], (double)ins[(j + 1) * AP_COLS + lane], a1);
      a2 = fma(crow[j + 2], (double)ins[(j + 2) * AP_COLS + lane], a2);
      a3 = fma(crow[j + 3], (double)ins[(j + 3) * AP_COLS + lane], a3);
    }
    for (; j < jend; ++j) a0 = fma(crow[j], (double)ins[j * AP_COLS + lane], a0);
    if (x < d) {
      const float o = (float)((a0 + a1) + (a2 + a3));
      const int64_t e = (int64_t)oi * d + x;
      OUT[e] = o;
      if (Wb) split_store(Wb, Wr, lo_off, e, o);  // the next pass's operand
    }
  }
}

static ppca_status apply_rows_small(Ctx* c, const double* C, int ldc, int rows, int m_in, const int* row_map,
                              bool lower, const float* IN, int64_t d, float* OUT, cudaStream_t st,
                              const WPrep* prep = nullptr) {
  static uint64_t attr = 0;
  if (first_on_device(&attr, c->device))
    cudaFuncSetAttribute(apply_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  // row blocks (multiples of 8 rows) until the grid covers the SMs: d = 1024 alone gives 32 CTAs
  const int64_t gx = ceil_div(d, (int64_t)AP_COLS);
  static const bool split = tune_env("PPCA_APPLY_SPLIT", 1) != 0;
  int rpc = rows;
  if (split && gx < c->sm_count) {
    const int gy = (int)std::min<int64_t>(ceil_div((int64_t)c->sm_count, gx), ceil_div((int64_t)rows, (int64_t)8));
    rpc = (int)ceil_div((int64_t)ceil_div((int64_t)rows, (int64_t)gy), (int64_t)8) * 8;
  }
  const unsigned gy = (unsigned)ceil_div((int64_t)rows, (int64_t)rpc);
  size_t smem = (size_t)rpc * m_in * sizeof(double) + (size_t)m_in * AP_COLS * sizeof(float);
  launch_pdl(apply_rows_kernel, dim3(dim3((unsigned)gx, gy)), dim3(256), smem, st, C, ldc, rows, m_in, row_map, lower, IN, d, OUT, rpc,
             prep ? prep->Wb : nullptr, prep ? prep->Wr : nullptr, prep ? prep->lo_off : (int64_t)0);
  PPCA_LAUNCH_CHECK(c, "apply_rows");
  return PPCA_OK;
}

constexpr int AT_COLS = 32;

template <int RPT>
__global__ void __launch_bounds__(256) apply_tiled_kernel(const double* __restrict__ C, int ldc, int rows, int m_in,
                                                          const int* __restrict__ row_map, bool lower,
                                                          const float* __restrict__ IN, int64_t d,
                                                          float* __restrict__ OUT) {
  pdl_enter();
  constexpr int RP = 32 * RPT, LDT = RP + 2;      // Cᵀ rows padded: 16-byte aligned, 4-way worst transposed store
  constexpr int PER = (128 * AT_COLS) / 256;      // staged IN values per thread (m_in ≤ 128)
  // [m_in][LDT] fp64, then IN staged as fp64 [m_in][2][8] double2 — (column pair p, column group cg): the
  // conversion runs once per staged value (16 per thread and chunk) instead of four per thread and j (fp32 → fp64
  // conversions issue at a quarter of the DFMA rate: as many pipe cycles as the 16 DFMAs they fed), and a quarter
  // warp's 16-byte loads of one pair are 128 contiguous bytes
  extern __shared__ __align__(16) double ct[];
  double* ins = ct + (size_t)m_in * LDT;
  copy_batched<8>(threadIdx.x, (int64_t)rows * m_in, 256,
                  [&](int64_t e) {
                    const int i = (int)(e / m_in), j = (int)(e % m_in);
                    return (!lower || j <= i) ? C[(int64_t)i * ldc + j] : 0.0;
                  },
                  [&](int64_t e, double v) { ct[(e % m_in) * LDT + e / m_in] = v; });
  for (int e = threadIdx.x; e < m_in * (RP - rows); e += 256) ct[(e / (RP - rows)) * LDT + rows + e % (RP - rows)] = 0.0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rg = lane >> 3, cg = lane & 7;
  // row sets: plain — warp w owns rows [4·RPT·w, 4·RPT·(w+1)); balanced (lower, RPT = 4) — warp w owns the 8-row
  // blocks w and 15 − w, so every warp (one per SM sub-partition pair) does the same triangular work
  const bool bal = lower && RPT == 4;
  int rows_t[RPT];
#pragma unroll
  for (int r = 0; r < RPT; ++r)
    rows_t[r] = bal ? (r < 2 ? 8 * warp + 2 * rg + r : 8 * (15 - warp) + 2 * rg + (r - 2)) : warp * 4 * RPT + rg * RPT + r;
  const int i0 = rows_t[0];
  const int jend = !lower ? m_in : bal ? min(m_in, 8 * (16 - warp)) : min(m_in, (warp + 1) * 4 * RPT);
  const int jsplit = bal ? min(jend, 8 * (warp + 1)) : jend;          // below it all RPT rows, above only the high ones
  const int64_t nchunks = (d + AT_COLS - 1) / AT_COLS;
  float nxt[PER];
  auto fetch = [&](int64_t ch) {
    const int64_t x0 = ch * AT_COLS;
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int e = threadIdx.x + 256 * u, j = e / AT_COLS;
      const int64_t x = x0 + e % AT_COLS;
      nxt[u] = (j < m_in && x < d) ? __ldg(IN + (int64_t)j * d + x) : 0.f;
    }
  };
  int64_t ch = blockIdx.x;
  if (ch < nchunks) fetch(ch);
  for (; ch < nchunks; ch += gridDim.x) {
    __syncthreads();                               // Cᵀ written / the previous chunk consumed
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int e = threadIdx.x + 256 * u;
      const int cc = e % AT_COLS;
      if (e < m_in * AT_COLS) ins[(e / AT_COLS) * AT_COLS + ((cc & 3) >> 1) * 16 + (cc >> 2) * 2 + (cc & 1)] = (double)nxt[u];
    }
    __syncthreads();
    if (ch + gridDim.x < nchunks) fetch(ch + gridDim.x);
    double acc[RPT][4];
#pragma unroll
    for (int r = 0; r < RPT; ++r)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[r][q] = 0.0;
#pragma unroll 4
    for (int j = 0; j < jsplit; ++j) {
      const double2 b01 = *reinterpret_cast<const double2*>(ins + j * AT_COLS + cg * 2);
      const double2 b23 = *reinterpret_cast<const double2*>(ins + j * AT_COLS + 16 + cg * 2);
      double a[RPT];
      if constexpr (RPT == 1) {
        a[0] = ct[j * LDT + i0];
      } else {
#pragma unroll
        for (int r = 0; r < RPT; r += 2) {        // row pairs are even-aligned: 16-byte aligned loads
          const double2 v = *reinterpret_cast<const double2*>(ct + j * LDT + rows_t[r]);
          a[r] = v.x;
          a[r + 1] = v.y;
        }
      }
      const double bb[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
      for (int r = 0; r < RPT; ++r)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[r][q] = fma(a[r], bb[q], acc[r][q]);
    }
    if constexpr (RPT == 4) {
#pragma unroll 4
      for (int j = jsplit; j < jend; ++j) {          // balanced lower: the high rows only
        const double2 b01 = *reinterpret_cast<const double2*>(ins + j * AT_COLS + cg * 2);
        const double2 b23 = *reinterpret_cast<const double2*>(ins + j * AT_COLS + 16 + cg * 2);
        const double2 v = *reinterpret_cast<const double2*>(ct + j * LDT + rows_t[2]);
        const double bb[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          acc[2][q] = fma(v.x, bb[q], acc[2][q]);
          acc[3][q] = fma(v.y, bb[q], acc[3][q]);
        }
      }
    }
    const int64_t x0 = ch * AT_COLS + cg * 4;
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const int i = rows_t[r];
      if (i >= rows) continue;
      const int oi = row_map ? row_map[i] : i;
      if (oi < 0) continue;
      float* o = OUT + (int64_t)oi * d;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (x0 + q < d) o[x0 + q] = (float)acc[r][q];
    }
  }
}

template <int RPT>
static void launch_apply_tiled(Ctx* c, const double* C, int ldc, int rows, int m_in, const int* row_map, bool lower,
                               const float* IN, int64_t d, float* OUT, cudaStream_t st) {
  const size_t smem = (size_t)m_in * (32 * RPT + 2) * sizeof(double) + (size_t)m_in * AT_COLS * sizeof(double);
  static uint64_t attr = 0;
  if (first_on_device(&attr, c->device))
    cudaFuncSetAttribute(apply_tiled_kernel<RPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int64_t nchunks = ceil_div(d, (int64_t)AT_COLS);
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(nchunks, c->sm_count));
  launch_pdl(apply_tiled_kernel<RPT>, dim3(grid), dim3(256), smem, st, C, ldc, rows, m_in, row_map, lower, IN, d, OUT);
}

static bool apply_small(const Ctx* c, int64_t d) { return ceil_div(d, (int64_t)AT_COLS) < 2 * c->sm_count; }

bool wprep_fusable(const Ctx* c, int m, int mp, int64_t d) { return m == mp && m <= 128 && apply_small(c, d); }

static ppca_status apply_rows(Ctx* c, const double* C, int ldc, int rows, int m_in, const int* row_map,
                              bool lower, const float* IN, int64_t d, float* OUT, cudaStream_t st,
                              const WPrep* prep = nullptr) {
  if (rows < 1 || m_in < 1 || d < 1) return PPCA_OK;
  if (rows > 128 || m_in > 128) return set_error(c, PPCA_ERR_UNSUPPORTED, "apply: %d x %d > 128", rows, m_in);
  if (apply_small(c, d))
    return apply_rows_small(c, C, ldc, rows, m_in, row_map, lower, IN, d, OUT, st, prep);
  if (prep) return set_error(c, PPCA_ERR_UNSUPPORTED, "apply: fused operand split needs the short-d kernel");
  if (rows <= 32) launch_apply_tiled<1>(c, C, ldc, rows, m_in, row_map, lower, IN, d, OUT, st);
  else if (rows <= 64) launch_apply_tiled<2>(c, C, ldc, rows, m_in, row_map, lower, IN, d, OUT, st);
  else launch_apply_tiled<4>(c, C, ldc, rows, m_in, row_map, lower, IN, d, OUT, st);
  PPCA_LAUNCH_CHECK(c, "apply_rows");
  return PPCA_OK;
}

// L⁻¹ of chol(G) (one CTA, fp64) on stream st; no drops (a non-positive pivot flags DEV_COLLAPSE)
ppca_status chol_inv_on(Ctx* c, const double* G, int m, double* Linv, int* row_map, int* m_out, cudaStream_t st) {
  static uint64_t attr = 0;
  if (first_on_device(&attr, c->device)) {
    cudaFuncSetAttribute(chol_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  }
  if (m <= 2 * CF_M && g_chol_reg) {
    launch_chol_inv_reg(G, m, Linv, row_map, m_out, c->d_err, st);
  } else {
    const size_t smem = chol_inv_smem(m);
    launch_pdl(chol_inv_kernel, dim3(1), dim3(256), smem, st, G, m, 0.0, Linv, row_map, m_out, c->d_err);
  }
  PPCA_LAUNCH_CHECK(c, "chol_inv");
  return PPCA_OK;
}

// OUT = L · IN for a lower-triangular fp64 L (m × m), IN/OUT [m][d] fp32, fp64 accumulation
ppca_status apply_lower_on(Ctx* c, const double* L, int m, const float* IN, int64_t d, float* OUT, cudaStream_t st) {
  return apply_rows(c, L, m, m, m, nullptr, true, IN, d, OUT, st);
}

// ============================================================================ CholQR2
ppca_status cholqr2(Ctx* c, float* W, int m, int64_t d, double drop_tol, int* m_out) {
  return cholqr(c, W, W, m, d, drop_tol, m_out, 2);
}

// W = Q-factor of the rows of Zin (positive diag R).  One pass is exact up to ε64·κ(Zin)² in fp64
// (the Gram, Cholesky and apply are fp64); a second pass restores orthonormality for ill-conditioned
// inputs (the refine path).
ppca_status cholqr(Ctx* c, const float* Zin, float* W, int m, int64_t d, double drop_tol, int* m_out, int passes,
                   bool gram_ready, const WPrep* prep) {
  double* G = (double*)scratch(c, S_GRAM, (size_t)m * m * sizeof(double));
  double* Linv = (double*)scratch(c, S_SMALL, (size_t)m * m * sizeof(double) + 2 * m * sizeof(int) + 64);
  int* row_map = (int*)(Linv + (size_t)m * m);
  int* d_mout = row_map + m;
  float* T = (float*)scratch(c, S_W2, (size_t)m * d * sizeof(float));
  if (!G || !Linv || !T) return set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
  static uint64_t attr = 0;
  if (first_on_device(&attr, c->device)) {
    cudaFuncSetAttribute(chol_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  }
  const size_t smem = chol_inv_smem(m);
  if (Zin != W && passes == 1 && drop_tol <= 0.0) {
    if (!gram_ready) PPCA_TRY(vec_gram(c, Zin, m, d, G));
    if (m <= 2 * CF_M && g_chol_reg)
      launch_chol_inv_reg(G, m, Linv, row_map, d_mout, c->d_err, c->stream);
    else
      launch_pdl(chol_inv_kernel, dim3(1), dim3(256), smem, c->stream, G, m, 0.0, Linv, row_map, d_mout, c->d_err);
    PPCA_LAUNCH_CHECK(c, "chol_inv");
    PPCA_TRY(apply_rows(c, Linv, m, m, m, nullptr, true, Zin, d, W, c->stream, prep));
    if (m_out) *m_out = m;
    return PPCA_OK;
  }
  if (prep) return set_error(c, PPCA_ERR_UNSUPPORTED, "cholqr: fused operand split on the one-pass path only");
  if (Zin != W)
    PPCA_TRY(check_cuda(c, cudaMemcpyAsync(W, Zin, (size_t)m * d * sizeof(float), cudaMemcpyDeviceToDevice, c->stream),
                        "copy Z"));
  for (int pass = 0; pass < passes; ++pass) {
    PPCA_TRY(vec_gram(c, W, m, d, G));
    const double dt = pass == 0 ? drop_tol : 0.0;
    if (dt <= 0.0 && m <= 2 * CF_M && g_chol_reg)
      launch_chol_inv_reg(G, m, Linv, row_map, d_mout, c->d_err, c->stream);
    else
      launch_pdl(chol_inv_kernel, dim3(1), dim3(256), smem, c->stream, G, m, dt, Linv, row_map, d_mout, c->d_err);
    PPCA_LAUNCH_CHECK(c, "chol_inv");
    if (pass == 0 && drop_tol > 0.0) {
      int h_m = m;
      PPCA_TRY(check_cuda(c, cudaMemcpyAsync(&h_m, d_mout, sizeof(int), cudaMemcpyDeviceToHost, c->stream),
                          "copy m_out"));
      PPCA_TRY(check_cuda(c, cudaStreamSynchronize(c->stream), "sync m_out"));
      PPCA_TRY(apply_rows(c, Linv, m, m, m, row_map, true, W, d, T, c->stream));
      PPCA_TRY(check_cuda(c, cudaMemcpyAsync(W, T, (size_t)h_m * d * sizeof(float), cudaMemcpyDeviceToDevice,
                                             c->stream), "copy W"));
      m = h_m;
      if (m_out) *m_out = h_m;
      if (m == 0) return set_error(c, PPCA_ERR_SUBSPACE_COLLAPSE, "all vectors collapsed");
      continue;
    }
    PPCA_TRY(apply_rows(c, Linv, m, m, m, nullptr, true, W, d, T, c->stream));
    PPCA_TRY(check_cuda(c, cudaMemcpyAsync(W, T, (size_t)m * d * sizeof(float), cudaMemcpyDeviceToDevice,
                                           c->stream), "copy W"));
  }
  if (m_out && drop_tol <= 0.0) *m_out = m;
  return PPCA_OK;
}

// ============================================================================ Rayleigh–Ritz (one CTA)
#include "ritz.cuh"

ppca_status ritz_debug_clocks(unsigned long long* out8) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out8, ritz::g_ritz_clk, 8 * sizeof(unsigned long long));
  cudaMemcpyFromSymbol(out8 + 8, g_chol_clk, 8 * sizeof(unsigned long long));
  return PPCA_OK;
}

static const int g_ritz_opt = tune_env("PPCA_RITZ_OPT", 5);   // ritz_values_kernel's opt bits (ritz.cuh)
ppca_status ritz_solve(Ctx* c, const double* S, const double* Bm, int m, double* theta_dev, double* R_dev,
                       cudaStream_t stream, int top) {
  double* scr = (double*)scratch(c, S_EVAL, (size_t)2 * m * m * sizeof(double));
  if (!scr) return set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
  static uint64_t attr = 0;
  if (first_on_device(&attr, c->device)) {
    cudaFuncSetAttribute(ritz::ritz_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, 208 * 1024);
    cudaFuncSetAttribute(ritz::ritz_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 208 * 1024);
  }
  static int jacobi = -1;                         // PPCA_RITZ_JACOBI=1: the Jacobi solver for vectors too
  if (jacobi < 0) jacobi = tune_env("PPCA_RITZ_JACOBI", 0);
  if (!R_dev || (m <= 64 && !jacobi)) {           // tridiagonalisation + multisection (+ inverse iteration)
    static uint64_t vattr = 0;
    if (first_on_device(&vattr, c->device)) {
      cudaFuncSetAttribute(ritz::ritz_values_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);   // + 32 KB static
    }
    const size_t vsm = (R_dev && m <= 64) ? ritz::vectors_smem_bytes(m) : ritz::values_smem_bytes(m);
    ritz::ritz_values_kernel<<<1, 512, vsm, stream>>>(S, Bm, m, scr, scr + (size_t)m * m, theta_dev, c->d_err, R_dev,
                                                      R_dev ? top : 0, g_ritz_opt);
    PPCA_LAUNCH_CHECK(c, "ritz_values_kernel");
    return PPCA_OK;
  }
  const size_t smem = ritz::smem_bytes(m);
  if (m <= 64)
    ritz::ritz_kernel<double><<<1, 512, smem, stream>>>(S, Bm, m, scr, scr + (size_t)m * m, theta_dev, R_dev, c->d_err);
  else
    ritz::ritz_kernel<float><<<1, 512, smem, stream>>>(S, Bm, m, scr, scr + (size_t)m * m, theta_dev, R_dev, c->d_err);
  PPCA_LAUNCH_CHECK(c, "ritz_kernel");
  return PPCA_OK;
}

// ============================================================================ sign convention, lift
__global__ void sign_rows_kernel(float* __restrict__ E, int64_t d) {
  float* row = E + (int64_t)blockIdx.x * d;
  float best = -1.f;
  int64_t bi = 0;
  for (int64_t x = threadIdx.x; x < d; x += blockDim.x) {
    float a = fabsf(row[x]);
    if (a > best) { best = a; bi = x; }        // first max within the thread's stride
  }
  __shared__ float sb[32];
  __shared__ long long si[32];
  // warp argmax (ties → lower index)
  for (int o = 16; o > 0; o >>= 1) {
    float ob = __shfl_xor_sync(0xffffffffu, best, o);
    long long oi = __shfl_xor_sync(0xffffffffu, (long long)bi, o);
    if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
  }
  if ((threadIdx.x & 31) == 0) { sb[threadIdx.x >> 5] = best; si[threadIdx.x >> 5] = bi; }
  __syncthreads();
  __shared__ float sgn;
  if (threadIdx.x == 0) {
    float b = sb[0];
    long long i = si[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      if (sb[w] > b || (sb[w] == b && si[w] < i)) { b = sb[w]; i = si[w]; }
    sgn = row[i] < 0.f ? -1.f : 1.f;
  }
  __syncthreads();
  if (sgn < 0.f)
    for (int64_t x = threadIdx.x; x < d; x += blockDim.x) row[x] = -row[x];
}

// Very long rows (d ≥ 2^20, the huge-d regime): one block per row would stream megabytes alone, so the rows are
// cut into ROWSLICES slices — partial (|max|, index) per slice, then every slice block reduces its row's partials
// (ties → lower index, so the order does not matter) and flips its slice.  Shorter rows keep sign_rows_kernel.
constexpr int64_t kLongRow = int64_t(1) << 20;
constexpr int ROWSLICES = 64;
__global__ void sign_part_kernel(const float* __restrict__ E, int64_t d, float* __restrict__ pb,
                                 long long* __restrict__ pi) {
  const int64_t L = (d + ROWSLICES - 1) / ROWSLICES, x0 = blockIdx.x * L, x1 = min(d, x0 + L);
  const float* row = E + (int64_t)blockIdx.y * d;
  float best = -1.f;
  long long bi = x0;
  for (int64_t x = x0 + threadIdx.x; x < x1; x += blockDim.x) {
    const float a = fabsf(row[x]);
    if (a > best) { best = a; bi = x; }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const float ob = __shfl_xor_sync(0xffffffffu, best, o);
    const long long oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
  }
  __shared__ float sb[32];
  __shared__ long long si[32];
  if ((threadIdx.x & 31) == 0) { sb[threadIdx.x >> 5] = best; si[threadIdx.x >> 5] = bi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      if (sb[w] > best || (sb[w] == best && si[w] < bi)) { best = sb[w]; bi = si[w]; }
    pb[blockIdx.y * ROWSLICES + blockIdx.x] = best;
    pi[blockIdx.y * ROWSLICES + blockIdx.x] = bi;
  }
}
__global__ void sign_apply_kernel(float* __restrict__ E, int64_t d, const float* __restrict__ pb,
                                  const long long* __restrict__ pi) {
  __shared__ float sgn;
  float* row = E + (int64_t)blockIdx.y * d;
  if (threadIdx.x == 0) {
    float b = pb[blockIdx.y * ROWSLICES];
    long long i = pi[blockIdx.y * ROWSLICES];
    for (int s = 1; s < ROWSLICES; ++s) {
      const float ob = pb[blockIdx.y * ROWSLICES + s];
      const long long oi = pi[blockIdx.y * ROWSLICES + s];
      if (ob > b || (ob == b && oi < i)) { b = ob; i = oi; }
    }
    sgn = row[i] < 0.f ? -1.f : 1.f;
  }
  __syncthreads();
  const int64_t L = (d + ROWSLICES - 1) / ROWSLICES, x0 = blockIdx.x * L, x1 = min(d, x0 + L);
  if (sgn < 0.f)
    for (int64_t x = x0 + threadIdx.x; x < x1; x += blockDim.x) row[x] = -row[x];
}

ppca_status lift_rows(Ctx* c, const double* R, int ldr, const float* W, int m, int k, int64_t d, float* E,
                      bool apply_sign, cudaStream_t stream) {
  PPCA_TRY(apply_rows(c, R, ldr, k, m, nullptr, false, W, d, E, stream));
  if (apply_sign && d >= kLongRow) {
    uint8_t* buf = (uint8_t*)scratch(c, S_SIGN, (size_t)k * ROWSLICES * (sizeof(float) + sizeof(long long)));
    if (!buf) return set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
    long long* pi = reinterpret_cast<long long*>(buf);
    float* pb = reinterpret_cast<float*>(pi + (size_t)k * ROWSLICES);
    sign_part_kernel<<<dim3(ROWSLICES, k), 256, 0, stream>>>(E, d, pb, pi);
    PPCA_LAUNCH_CHECK(c, "sign_part");
    sign_apply_kernel<<<dim3(ROWSLICES, k), 256, 0, stream>>>(E, d, pb, pi);
    PPCA_LAUNCH_CHECK(c, "sign_apply");
  } else if (apply_sign) {
    sign_rows_kernel<<<k, 256, 0, stream>>>(E, d);
    PPCA_LAUNCH_CHECK(c, "sign_rows");
  }
  return PPCA_OK;
}

// ============================================================================ init / normalise
__global__ void init_rows_kernel(uint64_t seed, float* __restrict__ W, int m, int64_t d) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)m * d) return;
  W[e] = (float)gaussian_elt(seed, 6u, (uint64_t)e);
}

__global__ void row_norm_kernel(const float* __restrict__ W, int64_t d, double* __restrict__ nrm) {
  const float* row = W + (int64_t)blockIdx.x * d;
  double s = 0.0;
  for (int64_t x = threadIdx.x; x < d; x += blockDim.x) s += (double)row[x] * row[x];
  s = warp_sum(s);
  __shared__ double red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    nrm[blockIdx.x] = sqrt(t);
  }
}

__global__ void scale_rows_kernel(float* __restrict__ W, int m, int64_t d, const double* __restrict__ nrm,
                                  int* d_err) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)m * d) return;
  double n = nrm[e / d];
  if (!(n > 1e-300)) {
    atomicOr(d_err, DEV_DEGENERATE);
    return;
  }
  double v = (double)W[e] / n;
  if (!isfinite(v)) atomicOr(d_err, DEV_NONFINITE);
  W[e] = (float)v;
}

// long rows (d ≥ 2^20): partial squared norms per slice, summed in slice order
__global__ void row_norm_part_kernel(const float* __restrict__ W, int64_t d, double* __restrict__ part) {
  const int64_t L = (d + ROWSLICES - 1) / ROWSLICES, x0 = blockIdx.x * L, x1 = min(d, x0 + L);
  const float* row = W + (int64_t)blockIdx.y * d;
  double s = 0.0;
  for (int64_t x = x0 + threadIdx.x; x < x1; x += blockDim.x) s += (double)row[x] * row[x];
  s = warp_sum(s);
  __shared__ double red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    part[blockIdx.y * ROWSLICES + blockIdx.x] = t;
  }
}
__global__ void row_norm_finish_kernel(const double* __restrict__ part, int m, double* __restrict__ nrm) {
  const int j = threadIdx.x;
  if (j >= m) return;
  double t = 0.0;
  for (int s = 0; s < ROWSLICES; ++s) t += part[j * ROWSLICES + s];
  nrm[j] = sqrt(t);
}

ppca_status normalize_rows(Ctx* c, float* W, int m, int64_t d) {
  double* nrm = (double*)scratch(c, S_ROWRED, (size_t)PPCA_MAX_M * (ROWSLICES + 1) * sizeof(double));
  if (!nrm) return set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
  if (d >= kLongRow) {
    double* part = nrm + PPCA_MAX_M;
    row_norm_part_kernel<<<dim3(ROWSLICES, m), 256, 0, c->stream>>>(W, d, part);
    PPCA_LAUNCH_CHECK(c, "row_norm_part");
    row_norm_finish_kernel<<<1, 128, 0, c->stream>>>(part, m, nrm);
  } else {
    row_norm_kernel<<<m, 256, 0, c->stream>>>(W, d, nrm);
  }
  PPCA_LAUNCH_CHECK(c, "row_norm");
  scale_rows_kernel<<<(unsigned)ceil_div((int64_t)m * d, 256), 256, 0, c->stream>>>(W, m, d, nrm, c->d_err);
  PPCA_LAUNCH_CHECK(c, "scale_rows");
  return PPCA_OK;
}

ppca_status init_rows(Ctx* c, uint64_t seed, float* W, int m, int64_t d) {
  init_rows_kernel<<<(unsigned)ceil_div((int64_t)m * d, 256), 256, 0, c->stream>>>(seed, W, m, d);
  PPCA_LAUNCH_CHECK(c, "init_rows");
  return normalize_rows(c, W, m, d);
}

// ============================================================================ priming updates
// Oja:  T = tril(P)·W  (apply), then elementwise  G = Q − T,  v ← μv + G,  W ← W + α(G + μv).
__global__ void oja_elementwise_kernel(const float* __restrict__ Q, const float* __restrict__ T,
                                       float* __restrict__ W, float* __restrict__ vel, int64_t count,
                                       double alpha, double mu, int* d_err) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= count) return;
  double g = (double)Q[e] - (double)T[e];
  double v = mu * (double)vel[e] + g;
  double w = (double)W[e] + alpha * (g + mu * v);
  if (!isfinite(w)) atomicOr(d_err, DEV_NONFINITE);
  vel[e] = (float)v;
  W[e] = (float)w;
}

ppca_status oja_update(Ctx* c, const float* Q, const double* P, float* W, float* vel, int m, int64_t d,
                       double alpha, double mu) {
  float* T = (float*)scratch(c, S_W3, (size_t)m * d * sizeof(float));
  PPCA_TRY(apply_rows(c, P, m, m, m, nullptr, true, W, d, T, c->stream));
  int64_t count = (int64_t)m * d;
  oja_elementwise_kernel<<<(unsigned)ceil_div(count, 256), 256, 0, c->stream>>>(Q, T, W, vel, count, alpha, mu,
                                                                                c->d_err);
  PPCA_LAUNCH_CHECK(c, "oja_elementwise");
  return PPCA_OK;
}

// EigenGame coefficients from A (m×m): Cf[j][i] = A_ji / A_ii (i < j), twoU[j] = 2(A_jj − Σ_{i<j} A_ji²/A_ii).
// One CTA: diagonal reciprocals in shared memory, then warp-per-j rows (lanes over i, fixed-order sums).
__global__ void __launch_bounds__(256) eg_coeff_kernel(const double* __restrict__ A, int m, double* __restrict__ Cf,
                                                       double* __restrict__ twoU, int* d_err) {
  __shared__ double rdiag[PPCA_MAX_M];
  __shared__ double amax;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp == 0) {
    double mx = 0.0;
    for (int i = lane; i < m; i += 32) mx = fmax(mx, A[i * m + i]);
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) amax = mx;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    double aii = A[i * m + i];
    if (!(aii > 1e-12 * amax)) {
      atomicOr(d_err, DEV_DEGENERATE);
      aii = 1.0;
    }
    rdiag[i] = 1.0 / aii;
  }
  __syncthreads();
  for (int j = warp; j < m; j += blockDim.x >> 5) {
    double part = 0.0;
    for (int i = lane; i < m; i += 32) {
      double cf = 0.0;
      if (i < j) {
        const double aji = A[j * m + i];
        cf = aji * rdiag[i];
        part += aji * cf;
      }
      Cf[j * m + i] = cf;
    }
    part = warp_sum(part);
    if (lane == 0) twoU[j] = 2.0 * (A[j * m + j] - part);
  }
}

__global__ void eg_elementwise_kernel(const float* __restrict__ MV, const float* __restrict__ T,
                                      const double* __restrict__ twoU, float* __restrict__ V,
                                      float* __restrict__ vel, int64_t d, int64_t count, double alpha,
                                      double mu, int* d_err) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= count) return;
  int64_t j = e / d;
  double r = 2.0 * (double)MV[e] - 2.0 * (double)T[e] - twoU[j] * (double)V[e];
  double v = mu * (double)vel[e] + r;
  double w = (double)V[e] + alpha * (r + mu * v);
  if (!isfinite(w)) atomicOr(d_err, DEV_NONFINITE);
  vel[e] = (float)v;
  V[e] = (float)w;
}

constexpr int EG_XC = 32;
constexpr int EG_ZPMAX = 16;    // row-group partials of Z summed while staging (the window pass's nrg ≤ 16)
#ifdef PPCA_EXPERIMENTS
__device__ unsigned long long g_eg_clk[8];          // phase stamps of CTA 0 (experiment builds)
#define EG_STAMP(i) do { if (blockIdx.x == 0 && threadIdx.x == 0) g_eg_clk[i] = clock64(); } while (0)
#else
#define EG_STAMP(i) do { } while (0)
#endif
// MV of this chunk into mvs[j][xl]: from the reduced MV, or (Zp != null) straight from the tensor-core window
// pass's row-group partials Zp[g][x][mp] — summed in g order in fp64 and rounded to fp32 exactly as the
// reduction kernel (reduce_zp) would have stored Z, so the result is bitwise the same without that launch
__device__ __forceinline__ void eg_stage_mv(const float* __restrict__ MV, const float* __restrict__ Zp, int64_t nrg,
                                            int64_t dpad, int mp, int m, int64_t d, int64_t x0, double* mvs) {
  const int tid = threadIdx.x;
  if (!Zp) {
    copy_batched<8>(tid, (int64_t)m * EG_XC, blockDim.x,
                    [&](int64_t e) {
                      const int64_t x = x0 + e % EG_XC;
                      return MV[(e / EG_XC) * d + (x < d ? x : d - 1)];
                    },
                    [&](int64_t e, float v) { mvs[e] = (double)v; });
    return;
  }
  const int q4 = mp >> 2;
  const int64_t gs = dpad * mp / 4;
  auto store = [&](int it, double a0, double a1, double a2, double a3) {
    const int xl = it / q4, j4 = (it % q4) * 4;
    if (j4 < m) mvs[j4 * EG_XC + xl] = (double)(float)a0;
    if (j4 + 1 < m) mvs[(j4 + 1) * EG_XC + xl] = (double)(float)a1;
    if (j4 + 2 < m) mvs[(j4 + 2) * EG_XC + xl] = (double)(float)a2;
    if (j4 + 3 < m) mvs[(j4 + 3) * EG_XC + xl] = (double)(float)a3;
  };
  auto src_of = [&](int it) {
    const int xl = it / q4, j4 = (it % q4) * 4;
    const int64_t x = min(x0 + xl, d - 1);
    return reinterpret_cast<const float4*>(Zp + x * mp + j4);
  };
  const int total = EG_XC * q4, nt = blockDim.x;
  if (nrg <= EG_ZPMAX / 2) {                          // two items per round, all their loads in flight
    for (int it = tid; it < total; it += 2 * nt) {
      const int it2 = it + nt;
      const float4* s1 = src_of(it);
      const float4* s2 = src_of(it2 < total ? it2 : it);
      float4 v1[EG_ZPMAX / 2], v2[EG_ZPMAX / 2];
#pragma unroll
      for (int g = 0; g < EG_ZPMAX / 2; ++g)
        if (g < nrg) {
          v1[g] = __ldg(s1 + g * gs);
          v2[g] = __ldg(s2 + g * gs);
        }
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0, b0 = 0.0, b1 = 0.0, b2 = 0.0, b3 = 0.0;
#pragma unroll
      for (int g = 0; g < EG_ZPMAX / 2; ++g)
        if (g < nrg) {
          a0 += (double)v1[g].x; a1 += (double)v1[g].y; a2 += (double)v1[g].z; a3 += (double)v1[g].w;
          b0 += (double)v2[g].x; b1 += (double)v2[g].y; b2 += (double)v2[g].z; b3 += (double)v2[g].w;
        }
      store(it, a0, a1, a2, a3);
      if (it2 < total) store(it2, b0, b1, b2, b3);
    }
    return;
  }
  for (int it = tid; it < total; it += nt) {
    const float4* src = src_of(it);
    float4 v[EG_ZPMAX];
#pragma unroll
    for (int g = 0; g < EG_ZPMAX; ++g)
      if (g < nrg) v[g] = __ldg(src + g * gs);
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
    for (int g = 0; g < EG_ZPMAX; ++g)
      if (g < nrg) {
        a0 += (double)v[g].x; a1 += (double)v[g].y; a2 += (double)v[g].z; a3 += (double)v[g].w;
      }
    store(it, a0, a1, a2, a3);
  }
}

// The whole EigenGame update in ONE cooperative kernel (the 5-launch sequence above costs ≈ 37 µs per C4 step,
// latency-bound): every CTA forms Cf = A_ji/A_ii and 2U from A itself (m×m, in shared memory — no barrier needed), then
// per 32-column chunk (lane = column, warp = rows j ≡ w mod 8): T_j = Σ_{i<j} Cf_ji·MV_i from a staged MV slab,
// r, Nesterov, V (unnormalised, rounded to fp32 as stored) and this chunk's Σ_x V_jx² per row; one grid
// barrier; then every CTA sums the chunks' row partials in chunk order (identical in all CTAs) and rescales
// its columns.  Same arithmetic as eg_coeff + apply_rows + eg_elementwise + normalize_rows.
// Latency: the first chunk's V, velocity and MV loads are issued before the m×m coefficient work (one round
// trip for all of them), and the row partials after the barrier are summed with every load in flight.
__global__ void __launch_bounds__(256) eg_update_kernel(const float* __restrict__ MV, const double* __restrict__ A,
                                                        float* __restrict__ V, float* __restrict__ vel, int m,
                                                        int64_t d, double alpha, double mu,
                                                        double* __restrict__ rowpart, int* d_err,
                                                        const float* __restrict__ Zp, int64_t nrg, int64_t dpad,
                                                        int mp, __nv_bfloat16* __restrict__ Wb, float* __restrict__ Wr,
                                                        int64_t lo_off) {
  pdl_enter();
  EG_STAMP(0);
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double egs[];
  double* Cf = egs;                                   // m × m
  double* twoU = Cf + (size_t)m * m;                  // m
  double* rdiag = twoU + m;                           // m
  double* nrm = rdiag + m;                            // m (reciprocal row norms)
  double* mvs = nrm + m;                             // m × EG_XC (MV as stored, fp32 values held in fp64)
  __shared__ double amax;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int64_t nchunks = (d + EG_XC - 1) / EG_XC;
  // this warp's V and velocity entries of the chunk (≤ PPCA_MAX_M / 8 rows per warp), in flight early
  float vpre[PPCA_MAX_M / 8], velpre[PPCA_MAX_M / 8];
  auto prefetch_vv = [&](int64_t ch) {
    const int64_t x = ch * EG_XC + lane;
#pragma unroll
    for (int q = 0; q < PPCA_MAX_M / 8; ++q) {
      const int j = warp + q * nw;
      const bool ok = j < m && x < d && ch < nchunks;
      vpre[q] = ok ? V[(int64_t)j * d + x] : 0.f;
      velpre[q] = ok ? vel[(int64_t)j * d + x] : 0.f;
    }
  };
  prefetch_vv(blockIdx.x);
  // coefficients (eg_coeff_kernel's arithmetic)
  if (warp == 0) {
    double mx = 0.0;
    for (int i = lane; i < m; i += 32) mx = fmax(mx, A[i * m + i]);
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) amax = mx;
  }
  copy_batched<16>(tid, (int64_t)m * m, blockDim.x, [&](int64_t e) { return A[e]; },
                   [&](int64_t e, double v) { Cf[e] = v; });
  if (blockIdx.x < nchunks) eg_stage_mv(MV, Zp, nrg, dpad, mp, m, d, (int64_t)blockIdx.x * EG_XC, mvs);
  __syncthreads();
  EG_STAMP(1);
  for (int i = tid; i < m; i += blockDim.x) {
    double aii = Cf[i * m + i];
    if (!(aii > 1e-12 * amax)) {
      if (blockIdx.x == 0) atomicOr(d_err, DEV_DEGENERATE);
      aii = 1.0;
    }
    rdiag[i] = 1.0 / aii;
  }
  __syncthreads();
  for (int j = warp; j < m; j += nw) {                // rows j: read A_j· (still in Cf), then overwrite with Cf_j·
    double part = 0.0;
    double cfv[PPCA_MAX_M / 32];
#pragma unroll
    for (int q = 0; q < PPCA_MAX_M / 32; ++q) {
      const int i = lane + 32 * q;
      double cf = 0.0;
      if (i < m && i < j) {
        const double aji = Cf[j * m + i];
        cf = aji * rdiag[i];
        part += aji * cf;
      }
      cfv[q] = cf;
    }
    part = warp_sum(part);
    const double ajj = Cf[j * m + j];
    __syncwarp();
#pragma unroll
    for (int q = 0; q < PPCA_MAX_M / 32; ++q) {
      const int i = lane + 32 * q;
      if (i < m) Cf[j * m + i] = cfv[q];
    }
    if (lane == 0) twoU[j] = 2.0 * (ajj - part);
  }
  __syncthreads();
  EG_STAMP(2);
  // update per column chunk; the squared row norms of this CTA's chunks accumulate in chunk order (lane 0 of
  // the row's warp) and leave as one partial per CTA
  double racc[PPCA_MAX_M / 8];
  float wkeep[PPCA_MAX_M / 8];
  const bool single = gridDim.x >= nchunks;          // one chunk per CTA: V stays in registers over the barrier
#pragma unroll
  for (int q = 0; q < PPCA_MAX_M / 8; ++q) {
    racc[q] = 0.0;
    wkeep[q] = 0.f;
  }
  for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const int64_t x0 = ch * EG_XC;
    if (ch != blockIdx.x) {                            // later chunks (grid < chunks): staged here
      eg_stage_mv(MV, Zp, nrg, dpad, mp, m, d, x0, mvs);
      prefetch_vv(ch);
      __syncthreads();
    }
    const int64_t x = x0 + lane;
#pragma unroll
    for (int q = 0; q < PPCA_MAX_M / 8; ++q) {
      const int j = warp + q * nw;
      if (j >= m) break;
      const double* cj = Cf + j * m;
      double t0 = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0;   // four chains, as the apply kernel; 8 loads in flight
      int i = 0;
      for (; i + 7 < j; i += 8) {
        double a[8], b[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          a[u] = cj[i + u];
          b[u] = mvs[(i + u) * EG_XC + lane];
        }
        t0 = fma(a[0], b[0], t0); t1 = fma(a[1], b[1], t1); t2 = fma(a[2], b[2], t2); t3 = fma(a[3], b[3], t3);
        t0 = fma(a[4], b[4], t0); t1 = fma(a[5], b[5], t1); t2 = fma(a[6], b[6], t2); t3 = fma(a[7], b[7], t3);
      }
      for (; i < j; ++i) t0 = fma(cj[i], mvs[i * EG_XC + lane], t0);
      const float tf = (float)((t0 + t1) + (t2 + t3));   // T as the apply kernel stores it (fp32)
      double sq = 0.0;
      if (x < d) {
        const int64_t e = (int64_t)j * d + x;
        const double r = 2.0 * mvs[j * EG_XC + lane] - 2.0 * (double)tf - twoU[j] * (double)vpre[q];
        const double v = mu * (double)velpre[q] + r;
        const double w = (double)vpre[q] + alpha * (r + mu * v);
        if (!isfinite(w)) atomicOr(d_err, DEV_NONFINITE);
        vel[e] = (float)v;
        const float wf = (float)w;
        if (single) wkeep[q] = wf;                     // rescaled from the register after the barrier
        else V[e] = wf;
        sq = (double)wf * wf;
      }
      sq = warp_sum(sq);
      racc[q] += sq;
    }
    __syncthreads();
  }
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < PPCA_MAX_M / 8; ++q) {
      const int j = warp + q * nw;
      if (j < m) rowpart[(int64_t)blockIdx.x * m + j] = racc[q];
    }
  }
  EG_STAMP(3);
  grid.sync();
  EG_STAMP(4);
  // row norms: thread (row j, slice s) sums the CTA partials c ≡ s (mod ns) in order (all loads in flight), the
  // slices are added in slice order — the same sums in every CTA; then this CTA's columns are rescaled
  {
    const int ns = (int)blockDim.x / m;                   // ≥ 2 for m ≤ 128
    const int j = threadIdx.x % m, sl = threadIdx.x / m;
    double* part = mvs;                                   // ns × m (the MV slab is free now)
    if (sl < ns)
      part[sl * m + j] = sum_in_order<32>(sl, (int64_t)gridDim.x, ns, [&](int64_t c1) { return rowpart[c1 * m + j]; });
    __syncthreads();
    if (threadIdx.x < m) {
      double s2 = 0.0;
      for (int q = 0; q < ns; ++q) s2 += part[q * m + threadIdx.x];
      const double n = sqrt(s2);
      if (!(n > 1e-300)) {
        if (blockIdx.x == 0) atomicOr(d_err, DEV_DEGENERATE);
        nrm[threadIdx.x] = 0.0;
      } else {
        nrm[threadIdx.x] = 1.0 / n;
      }
    }
  }
  __syncthreads();
  EG_STAMP(5);
  if (single) {
    const int64_t x = (int64_t)blockIdx.x * EG_XC + lane;
    if (x < d)
#pragma unroll
      for (int q = 0; q < PPCA_MAX_M / 8; ++q) {
        const int j = warp + q * nw;
        if (j >= m) break;
        const double v = nrm[j] > 0.0 ? (double)wkeep[q] * nrm[j] : (double)wkeep[q];
        if (!isfinite(v)) atomicOr(d_err, DEV_NONFINITE);
        const int64_t e = (int64_t)j * d + x;
        V[e] = (float)v;
        if (Wb) split_store(Wb, Wr, lo_off, e, (float)v);
      }
  } else {
    for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
      const int64_t x = ch * EG_XC + lane;
      if (x < d)
        for (int j = warp; j < m; j += nw) {
          const int64_t e = (int64_t)j * d + x;
          float vf = V[e];
          if (nrm[j] > 0.0) {
            const double v = (double)vf * nrm[j];
            if (!isfinite(v)) atomicOr(d_err, DEV_NONFINITE);
            vf = (float)v;
            V[e] = vf;
          }
          if (Wb) split_store(Wb, Wr, lo_off, e, vf);
        }
    }
  }
  EG_STAMP(6);
}

static bool eigengame_update_fused(Ctx* c, const float* MV, const double* A, float* V, float* vel, int m, int64_t d,
                                   double alpha, double mu, ppca_status* st, const WPrep* prep) {
  *st = PPCA_OK;
  const int64_t nchunks = ceil_div(d, (int64_t)EG_XC);
  const size_t smem = ((size_t)m * m + 3 * (size_t)m) * sizeof(double) +
                      std::max((size_t)m * EG_XC * sizeof(double), (size_t)256 * sizeof(double));
  static uint64_t attr = 0;
  if (first_on_device(&attr, c->device)) {
    cudaFuncSetAttribute(eg_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  }
  int per_sm = 0;
  if (smem > 200 * 1024 ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, eg_update_kernel, 256, smem) != cudaSuccess || per_sm < 1) {
    cudaGetLastError();
    return false;
  }
  const int grid = (int)std::min<int64_t>(nchunks, (int64_t)per_sm * c->sm_count);
  double* rowpart = (double*)scratch(c, S_ROWRED, (size_t)grid * m * sizeof(double));   // one partial per CTA
  if (!rowpart) {
    *st = set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
    return true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeCooperative;                       // one grid barrier: all CTAs co-resident
  at[0].val.cooperative = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // the launch overlaps the Q/P reduction's tail
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = g_pdl ? 2 : 1;
  // Z straight from the window pass's row-group partials when it left them (pass_defer_z)
  const float* Zp = nullptr;
  int64_t nrg = 0, dpad = 0;
  int mp = 0;
  if (c->zp_pending) {
    Zp = c->zp_part;
    nrg = c->zp_nrg;
    dpad = c->zp_dpad;
    mp = c->zp_mp;
  }
  cudaError_t e = cudaLaunchKernelEx(&cfg, eg_update_kernel, MV, A, V, vel, m, d, alpha, mu, rowpart, c->d_err, Zp,
                                     nrg, dpad, mp, prep ? prep->Wb : nullptr, prep ? prep->Wr : nullptr,
                                     prep ? prep->lo_off : (int64_t)0);
  if (e == cudaSuccess) c->zp_pending = false;
#ifdef PPCA_EXPERIMENTS
  static const int eg_clk = tune_env("PPCA_EG_CLK", 0);
  if (eg_clk && e == cudaSuccess) {
    unsigned long long t[8];
    cudaStreamSynchronize(c->stream);
    cudaMemcpyFromSymbol(t, g_eg_clk, sizeof(t));
    fprintf(stderr, "[eg_update] cycles: stage+A %llu  coeff %llu  chunk %llu  grid.sync %llu  norms %llu  rescale %llu\n",
            t[1] - t[0], t[2] - t[1], t[3] - t[2], t[4] - t[3], t[5] - t[4], t[6] - t[5]);
  }
#endif
  if (e == cudaErrorCooperativeLaunchTooLarge) {     // not all CTAs co-resident: the 5-launch sequence runs
    cudaGetLastError();
    return false;
  }
  ++c->launches;
  if (e != cudaSuccess) *st = check_cuda(c, e, "eg_update_kernel");
  return true;
}

ppca_status eigengame_update(Ctx* c, const float* MV, const double* A, float* V, float* vel, int m, int64_t d,
                             double alpha, double mu, const WPrep* prep, bool* prep_done) {
  static int multi = -1;                          // PPCA_EG_MULTI=1: the 5-launch sequence (comparison)
  if (multi < 0) multi = tune_env("PPCA_EG_MULTI", 0);
  if (prep_done) *prep_done = false;
  if (!multi) {
    ppca_status st;
    if (eigengame_update_fused(c, MV, A, V, vel, m, d, alpha, mu, &st, prep)) {
      if (prep_done) *prep_done = prep != nullptr && st == PPCA_OK;
      return st;
    }
  }
  PPCA_TRY(pass_reduce_deferred_z(c, const_cast<float*>(MV)));   // the multi-launch sequence reads Z itself
  double* Cf = (double*)scratch(c, S_SMALL, (size_t)m * m * sizeof(double) + (size_t)m * sizeof(double) + 64);
  double* twoU = Cf + (size_t)m * m;
  float* T = (float*)scratch(c, S_W3, (size_t)m * d * sizeof(float));
  eg_coeff_kernel<<<1, 256, 0, c->stream>>>(A, m, Cf, twoU, c->d_err);
  PPCA_LAUNCH_CHECK(c, "eg_coeff");
  PPCA_TRY(apply_rows(c, Cf, m, m, m, nullptr, false, MV, d, T, c->stream));
  int64_t count = (int64_t)m * d;
  eg_elementwise_kernel<<<(unsigned)ceil_div(count, 256), 256, 0, c->stream>>>(MV, T, twoU, V, vel, d, count,
                                                                               alpha, mu, c->d_err);
  PPCA_LAUNCH_CHECK(c, "eg_elementwise");
  return normalize_rows(c, V, m, d);
}

// ============================================================================ eval dots
__global__ void row_dots_kernel(const float* __restrict__ E, const float* __restrict__ T, int64_t d,
                                double* __restrict__ out) {
  const float* a = E + (int64_t)blockIdx.x * d;
  const float* b = T + (int64_t)blockIdx.x * d;
  double s = 0.0;
  for (int64_t x = threadIdx.x; x < d; x += blockDim.x) s += (double)a[x] * b[x];
  s = warp_sum(s);
  __shared__ double red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    out[blockIdx.x] = t;
  }
}

// res[i] = ‖Z_i − θ_i E_i‖ in fp64 (Z_i = (XᵀX e_i)ᵀ), one CTA per vector
__global__ void ritz_resid_kernel(const float* __restrict__ Z, const float* __restrict__ E,
                                  const double* __restrict__ theta, int64_t d, double* __restrict__ out) {
  const float* z = Z + (int64_t)blockIdx.x * d;
  const float* e = E + (int64_t)blockIdx.x * d;
  const double th = theta[blockIdx.x];
  double s = 0.0;
  for (int64_t x = threadIdx.x; x < d; x += blockDim.x) {
    const double r = (double)z[x] - th * (double)e[x];
    s = fma(r, r, s);
  }
  s = warp_sum(s);
  __shared__ double red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    out[blockIdx.x] = sqrt(t);
  }
}

ppca_status ritz_resid(Ctx* c, const float* Z, const float* E, const double* theta, int k, int64_t d, double* res) {
  ritz_resid_kernel<<<k, 256, 0, c->stream>>>(Z, E, theta, d, res);
  PPCA_LAUNCH_CHECK(c, "ritz_resid");
  return PPCA_OK;
}

// Z_i ← Z_i − θ_i E_i in place (fp32 result of an fp64 difference)
__global__ void resid_rows_kernel(float* __restrict__ Z, const float* __restrict__ E, const double* __restrict__ theta,
                                  int64_t d) {
  float* z = Z + (int64_t)blockIdx.y * d;
  const float* e = E + (int64_t)blockIdx.y * d;
  const double th = theta[blockIdx.y];
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < d; x += (int64_t)gridDim.x * blockDim.x)
    z[x] = (float)((double)z[x] - th * (double)e[x]);
}

ppca_status resid_rows(Ctx* c, float* Z, const float* E, const double* theta, int k, int64_t d) {
  resid_rows_kernel<<<dim3((unsigned)std::min<int64_t>(ceil_div(d, 256), 64), (unsigned)k), 256, 0, c->stream>>>(Z, E, theta, d);
  PPCA_LAUNCH_CHECK(c, "resid_rows");
  return PPCA_OK;
}

ppca_status row_dots(Ctx* c, const float* E, const float* T, int k, int64_t d, double* dots) {
  row_dots_kernel<<<k, 256, 0, c->stream>>>(E, T, d, dots);
  PPCA_LAUNCH_CHECK(c, "row_dots");
  return PPCA_OK;
}

// ============================================================================ Proposition 3 checker (NEXT-4)
// PAPER.md §4.2 Prop. 3 (L293-302), reading R28.  Inputs: the stacked Gram
// G = [B; T][B; T]ᵀ (ld g = mm + upto; B = the operand rows of the pass, T = the true eigenvectors) and the
// projected Gram S = (XBᵀ)ᵀ(XBᵀ).  With L = chol(BBᵀ) the rows of L⁻¹B are an orthonormal basis of
// span B, the projected covariance in it is C = L⁻¹SL⁻ᵀ and π_S(t_i) has coordinates y_i = L⁻¹(Bt_i).
// Kernel 1 (one CTA): C, y_i, ‖y_i‖/‖t_i‖ and the identity (the Ritz solve's metric), all fp64 in global
// scratch (the m×m work is O(m³) ≈ 2 MFLOP — a diagnostic, not a hot path).
__global__ void __launch_bounds__(256) prop3_coords_kernel(const double* __restrict__ G, int g,
                                                           const double* __restrict__ S, int mm, int upto,
                                                           double* __restrict__ A, double* __restrict__ Linv,
                                                           double* __restrict__ T1, double* __restrict__ C,
                                                           double* __restrict__ I, double* __restrict__ Y,
                                                           double* __restrict__ ratio, double* __restrict__ diag0,
                                                           int* __restrict__ keep, int* d_err) {
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int e = tid; e < mm * mm; e += nt) {
    const int a = e / mm, b = e % mm;
    A[e] = G[(int64_t)a * g + b];
    I[e] = a == b ? 1.0 : 0.0;
  }
  __syncthreads();
  block_cholesky(A, mm, 0.0, keep, diag0, d_err, mm);
  block_lower_inverse(A, mm, keep, Linv, mm, mm);
  __syncthreads();
  for (int e = tid; e < mm * mm; e += nt) {           // T1 = S L⁻ᵀ
    const int a = e / mm, b = e % mm;
    double acc = 0.0;
    for (int q = 0; q <= b; ++q) acc = fma(S[a * mm + q], Linv[b * mm + q], acc);
    T1[e] = acc;
  }
  __syncthreads();
  for (int e = tid; e < mm * mm; e += nt) {           // C = L⁻¹ T1
    const int a = e / mm, b = e % mm;
    double acc = 0.0;
    for (int q = 0; q <= a; ++q) acc = fma(Linv[a * mm + q], T1[q * mm + b], acc);
    C[e] = acc;
  }
  for (int e = tid; e < upto * mm; e += nt) {         // y_i = L⁻¹ (B t_i)
    const int i = e / mm, a = e % mm;
    double acc = 0.0;
    for (int q = 0; q <= a; ++q) acc = fma(Linv[a * mm + q], G[(int64_t)q * g + mm + i], acc);
    Y[e] = acc;
  }
  __syncthreads();
  for (int i = tid; i < upto; i += nt) {
    double yy = 0.0;
    for (int a = 0; a < mm; ++a) yy = fma(Y[i * mm + a], Y[i * mm + a], yy);
    const double tt = G[(int64_t)(mm + i) * g + mm + i];
    ratio[i] = tt > 0.0 ? sqrt(yy / tt) : 0.0;
  }
}

// Kernel 2 (CTA i): Q = orthonormal basis of y_1 … y_{i−1} (modified Gram–Schmidt with one
// re-orthogonalisation, residual < 1e-10 dropped — warp 0, a vector in registers, shuffle dots), then
// M_i = P C P with P = I − QᵀQ as C − QᵀWᵀ − W Q + Z Q  (W = C Qᵀ, H = Q W, Z = Qᵀ H), without forming P.
constexpr int P3_VR = PPCA_MAX_M / 32;
__global__ void __launch_bounds__(256) prop3_project_kernel(const double* __restrict__ C,
                                                            const double* __restrict__ Y, int mm,
                                                            double* __restrict__ Qg, double* __restrict__ Wg,
                                                            double* __restrict__ Zg, double* __restrict__ Hg,
                                                            double* __restrict__ Mg) {
  const int i = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  const size_t off = (size_t)i * mm * mm;
  double* Q = Qg + off;   // nq × mm
  double* W = Wg + off;   // mm × nq
  double* Z = Zg + off;   // mm × nq
  double* M = Mg + off;
  double* H = Hg + off;   // nq × nq
  __shared__ int nq_s;
  if (tid < 32) {
    const int lane = tid;
    int nq = 0;
    for (int j = 0; j < i; ++j) {
      double w[P3_VR];
#pragma unroll
      for (int r = 0; r < P3_VR; ++r) {
        const int a = lane + 32 * r;
        w[r] = a < mm ? Y[j * mm + a] : 0.0;
      }
      for (int pass = 0; pass < 2; ++pass)
        for (int q = 0; q < nq; ++q) {
          double dot = 0.0;
#pragma unroll
          for (int r = 0; r < P3_VR; ++r) {
            const int a = lane + 32 * r;
            if (a < mm) dot = fma(Q[q * mm + a], w[r], dot);
          }
#pragma unroll
          for (int o = 16; o; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
#pragma unroll
          for (int r = 0; r < P3_VR; ++r) {
            const int a = lane + 32 * r;
            if (a < mm) w[r] = fma(-dot, Q[q * mm + a], w[r]);
          }
        }
      double nn = 0.0;
#pragma unroll
      for (int r = 0; r < P3_VR; ++r) nn = fma(w[r], w[r], nn);
#pragma unroll
      for (int o = 16; o; o >>= 1) nn += __shfl_xor_sync(0xffffffffu, nn, o);
      const double nrm = sqrt(nn);
      if (nrm >= 1e-10) {
#pragma unroll
        for (int r = 0; r < P3_VR; ++r) {
          const int a = lane + 32 * r;
          if (a < mm) Q[nq * mm + a] = w[r] / nrm;
        }
        ++nq;
      }
      __syncwarp();
    }
    if (lane == 0) nq_s = nq;
  }
  __syncthreads();
  const int nq = nq_s;
  for (int e = tid; e < mm * nq; e += nt) {            // W = C Qᵀ  (mm × nq)
    const int a = e / nq, r = e % nq;
    double acc = 0.0;
    for (int b = 0; b < mm; ++b) acc = fma(C[a * mm + b], Q[r * mm + b], acc);
    W[e] = acc;
  }
  __syncthreads();
  for (int e = tid; e < nq * nq; e += nt) {            // H = Q W  (nq × nq)
    const int r = e / nq, s2 = e % nq;
    double acc = 0.0;
    for (int b = 0; b < mm; ++b) acc = fma(Q[r * mm + b], W[b * nq + s2], acc);
    H[e] = acc;
  }
  __syncthreads();
  for (int e = tid; e < mm * nq; e += nt) {            // Z = Qᵀ H  (mm × nq)
    const int a = e / nq, s2 = e % nq;
    double acc = 0.0;
    for (int r = 0; r < nq; ++r) acc = fma(Q[r * mm + a], H[r * nq + s2], acc);
    Z[e] = acc;
  }
  __syncthreads();
  for (int e = tid; e < mm * mm; e += nt) {            // M = C − QᵀWᵀ − W Q + Z Q
    const int a = e / mm, b = e % mm;
    double acc = C[e];
    for (int r = 0; r < nq; ++r)
      acc += -Q[r * mm + a] * W[b * nq + r] - W[a * nq + r] * Q[r * mm + b] + Z[a * nq + r] * Q[r * mm + b];
    M[e] = acc;
  }
}

// Kernel 3 (warp i): ∠(u_i, y_i) for u_i = row 0 of R_i (the top eigenvector of M_i), via
// atan2(‖u − (u·ŷ)ŷ‖, |u·ŷ|) — accurate at tiny angles where acos is not.
__global__ void prop3_angle_kernel(const double* __restrict__ R, const double* __restrict__ Y, int mm,
                                   double* __restrict__ ang) {
  const int i = blockIdx.x, lane = threadIdx.x;
  const double* u = R + (size_t)i * mm * mm;
  const double* y = Y + (size_t)i * mm;
  double yy = 0.0, uy = 0.0;
  for (int a = lane; a < mm; a += 32) {
    yy = fma(y[a], y[a], yy);
    uy = fma(u[a], y[a], uy);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    yy += __shfl_xor_sync(0xffffffffu, yy, o);
    uy += __shfl_xor_sync(0xffffffffu, uy, o);
  }
  const double c = uy / sqrt(yy);                      // u·ŷ
  double ss = 0.0;
  for (int a = lane; a < mm; a += 32) {
    const double r = u[a] - c * y[a] / sqrt(yy);
    ss = fma(r, r, ss);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if (lane == 0) ang[i] = atan2(sqrt(ss), fabs(c));
}

ppca_status prop3_device(Ctx* c, const double* G, int g, const double* S, int mm, int upto, double* ratio_host,
                         double* angles_host) {
  const size_t m2 = (size_t)mm * mm;
  double* w = (double*)scratch(c, S_P3, (7 * m2 + (size_t)upto * (6 * m2 + 2 * mm + 2) + 2 * mm + 64) * sizeof(double));
  if (!w) return set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
  double *A = w, *Linv = A + m2, *T1 = Linv + m2, *C = T1 + m2, *I = C + m2, *Y = I + m2;
  double* ratio = Y + (size_t)upto * mm;
  double* ang = ratio + upto;
  double* Qg = ang + upto;
  double* Wg = Qg + upto * m2;
  double* Zg = Wg + upto * m2;
  double* Hg = Zg + upto * m2;
  double* Mg = Hg + upto * m2;
  double* Rg = Mg + upto * m2;
  double* theta = Rg + upto * m2;
  double* diag0 = theta + (size_t)upto * mm;
  int* keep = (int*)(diag0 + mm);
  prop3_coords_kernel<<<1, 256, 0, c->stream>>>(G, g, S, mm, upto, A, Linv, T1, C, I, Y, ratio, diag0, keep, c->d_err);
  PPCA_LAUNCH_CHECK(c, "prop3_coords");
  PPCA_TRY(check_cuda(c, cudaMemcpyAsync(ratio_host, ratio, upto * sizeof(double), cudaMemcpyDeviceToHost, c->stream),
                      "copy ratios"));
  PPCA_TRY(finish(c, "ppca_check_prop3"));
  for (int i = 0; i < upto; ++i)                       // DegenerateProjection
    if (!(ratio_host[i] >= 1e-10))
      return set_error(c, PPCA_ERR_DEGENERATE, "|pi_S(e_%d)| = %.3g |e_%d| < 1e-10", i + 1, ratio_host[i], i + 1);
  prop3_project_kernel<<<upto, 256, 0, c->stream>>>(C, Y, mm, Qg, Wg, Zg, Hg, Mg);
  PPCA_LAUNCH_CHECK(c, "prop3_project");
  for (int i = 0; i < upto; ++i)                       // the variance maximiser on each complement
    PPCA_TRY(ritz_solve(c, Mg + i * m2, I, mm, theta + (size_t)i * mm, Rg + i * m2, c->stream));
  prop3_angle_kernel<<<upto, 32, 0, c->stream>>>(Rg, Y, mm, ang);
  PPCA_LAUNCH_CHECK(c, "prop3_angle");
  PPCA_TRY(check_cuda(c, cudaMemcpyAsync(angles_host, ang, upto * sizeof(double), cudaMemcpyDeviceToHost, c->stream),
                      "copy angles"));
  return PPCA_OK;
}

}  // namespace ppca
