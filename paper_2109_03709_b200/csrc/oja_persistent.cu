// oja_persistent.cu — generalized-Oja priming with small minibatches in ONE cooperative kernel (§8 row a5).
//
// C2's step (b = 256 rows × d = 784, m = 32) moves 0.8 MB: at HBM speed ~0.1 µs, so a step made of separate
// launches (products, reductions, update) is latency bound.  Here every step of a call runs inside one
// persistent cooperative launch (one 256-thread CTA per SM), three grid-wide barriers per step:
//   phase 1  Y = X_b·Wᵀ          items of (RG rows × 8 components): the rows staged in shared memory as fp32,
//                                 warp per component j streaming W[j][·] (float4), warp-shuffle reduction
//   phase 2  Q = X_bᵀY           items of 8 columns: X and Y staged in shared memory as fp64, thread per
//                                 (component, row group) with 8 register accumulators, groups reduced in order
//            P = YᵀY             items of 8 upper-triangle 4×4 tiles × 32 row groups, reduced in order; fp64
//   phase 3  G = Q − tril(P)·W, v ← μv + G, W ← W + α(G + μv)   items of XC columns, thread per (column,
//                                 component), fp64; a CTA stages the old columns of W before overwriting them
// Numerics follow the multi-launch path (fp32 Y, fp64 products and update; readings
// R8-R10).  Single GPU only (an all-reduce between phases 2 and 3 would need device-side NCCL).
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace ppca {

constexpr int OJA_MAXM = 64;
constexpr int OJA_THREADS = 256;
constexpr int OJA_RG = 8;          // rows per phase-1 item (max)
constexpr int OJA_XROW = 64 * 1024; // phase-1 row staging budget (bytes)
constexpr int OJA_SMEM = 140 * 1024;

struct OjaParams {
  const void* X;
  int xdtype;           // ppca_dtype
  int64_t ld, n, d;
  int m, batch, rg, xc, rc;
  int64_t s0, steps;
  float* W;             // [m][d]
  float* vel;           // [m][d]
  float* Y;             // [batch][m] scratch
  double* Q;            // [d][m] scratch (x-major)
  double* P;            // [m][m] scratch
  double alpha, mu;
  int* err;
  unsigned long long* clk;   // optional phase timestamps of the first step (PPCA_OJA_CLK)
  int xvec;                  // X rows 16-byte aligned with d % 8 == 0: vector loads
  int wvec;                  // W rows 16-byte aligned (d % 4 == 0): float4 loads in phase 1
  int dbg;                   // timing experiments only (PPCA_OJA_DBG): 1 skip phase-2 staging, 2 skip phase-2
                             // math, 4 skip phase-1 chunk loop, 8 skip phase-3 body, 16 skip phase 1, 32 skip phase 2,
                             // 64 no next-window L2 prefetch
};

template <typename T>
__device__ __forceinline__ float oja_ld(const T* X, const OjaParams& p, int64_t r, int64_t x) {
  return load_rc(X, p.ld, r, x, p.d);
}

// eight consecutive elements X[row][xb..xb+8) as fp64, one or two 16-byte loads per plane (needs the
// host-checked alignment: 16-byte aligned rows, xb % 8 == 0, xb + 8 <= d)
__device__ __forceinline__ void load_row8(const float* X, const OjaParams& p, int64_t row, int64_t xb, double* o) {
  const float4* q = reinterpret_cast<const float4*>(X + row * p.ld + xb);
  const float4 a = q[0], b = q[1];
  o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w; o[4] = b.x; o[5] = b.y; o[6] = b.z; o[7] = b.w;
}
__device__ __forceinline__ float bf_lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float bf_hi(uint32_t u) { return __uint_as_float(u & 0xffff0000u); }
__device__ __forceinline__ void load_row8(const __nv_bfloat16* X, const OjaParams& p, int64_t row, int64_t xb,
                                          double* o) {
  const uint4 a = *reinterpret_cast<const uint4*>(X + row * p.ld + xb);
  const uint32_t w[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    o[2 * u] = bf_lo(w[u]);
    o[2 * u + 1] = bf_hi(w[u]);
  }
}
__device__ __forceinline__ void load_row8(const SplitF32* X, const OjaParams& p, int64_t row, int64_t xb, double* o) {
  const __nv_bfloat16* r = reinterpret_cast<const __nv_bfloat16*>(X + row * p.ld);
  const uint4 h = *reinterpret_cast<const uint4*>(r + xb);
  const uint4 l = *reinterpret_cast<const uint4*>(r + p.d + xb);
  const uint32_t wh[4] = {h.x, h.y, h.z, h.w}, wl[4] = {l.x, l.y, l.z, l.w};
#pragma unroll
  for (int u = 0; u < 4; ++u) {             // hi + lo in fp32, as load_rc does
    o[2 * u] = (double)(bf_lo(wh[u]) + bf_lo(wl[u]));
    o[2 * u + 1] = (double)(bf_hi(wh[u]) + bf_hi(wl[u]));
  }
}

__device__ __forceinline__ float W_old(const OjaParams& p, int l, int64_t x) { return p.W[(int64_t)l * p.d + x]; }

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// dst[e] = f(e) for e < count, sixteen independent loads in flight per thread before the stores
template <typename D, typename F>
__device__ __forceinline__ void stage16(D* dst, int count, F f) {
  for (int e0 = threadIdx.x; e0 < count; e0 += 16 * blockDim.x) {
    D v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {                // unconditional (clamped) loads: all sixteen in flight
      const int e = e0 + u * blockDim.x;
      v[u] = f(e < count ? e : count - 1);
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int e = e0 + u * blockDim.x;
      if (e < count) dst[e] = v[u];
    }
  }
}

template <typename T>
__device__ void oja_steps(const OjaParams& p, const T* __restrict__ X, uint8_t* smem) {
  cg::grid_group grid = cg::this_grid();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int m = p.m;
  const int64_t d = p.d, nb = (p.n + p.batch - 1) / p.batch, nbf = p.n / p.batch;
  const int xc = p.xc, rc = p.rc, rg = p.rg;
  const int nxc = (int)((d + xc - 1) / xc);
  const int mp = (m + 3) & ~3;
  const int nq8 = (int)((d + 7) / 8);
  const int nt4 = mp / 4, nup = nt4 * (nt4 + 1) / 2;   // 4×4 tiles per side, upper-triangle tiles
  const int npg = (nup + 7) / 8;
  const int njg = (m + 7) / 8;
  const bool clk = p.clk != nullptr && blockIdx.x == 0 && tid == 0;
  const bool bclk = p.clk != nullptr && tid == 0;
  for (int64_t st = p.s0; st < p.s0 + p.steps; ++st) {
    const int64_t blk = st % nb;
    const int64_t r0 = blk * p.batch;
    const int rows = (int)(blk < nbf ? p.batch : p.n - nbf * p.batch);
    const bool rec = clk && st == p.s0;
    if (rec) p.clk[0] = gtimer();
    // ---- phase 1: Y = X_b·Wᵀ; item = (group of rg rows, group of 8 components); warp w takes component
    //      j = 8·jg + w and all rows of the group; lane partial sums over x, then a shuffle reduction
    {
      float* Xr = reinterpret_cast<float*>(smem);       // [rg][d]
      const int nrg = (rows + rg - 1) / rg;
      const int nitems = (p.dbg & 16) ? 0 : nrg * njg;
      int staged = -1;
      for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
        const int rgi = it / njg, jg = it - rgi * njg;
        const int rr0 = rgi * rg;
        const int nr = rows - rr0 < rg ? rows - rr0 : rg;
        const int j = jg * 8 + warp;
        const float* wj = p.W + (int64_t)(j < m ? j : m - 1) * d;
        const int n4 = (int)(d / 4);
        float4 w[8];                                      // first batch of W[j][·] in flight during staging
        if (p.wvec) {
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int k = lane + 32 * u;
            w[u] = reinterpret_cast<const float4*>(wj)[k < n4 ? k : n4 - 1];
          }
        }
        if (staged != rgi && !(p.dbg & 128)) {           // the item's rows as fp32 (rows past the window: 0)
          __syncthreads();
          if (p.xvec) {
            const int per = (int)(d / 8), cnt = rg * per;
            for (int e0 = tid; e0 < cnt; e0 += 4 * OJA_THREADS) {   // four 8-element groups in flight
              double o[4][8];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int e = min(e0 + u * OJA_THREADS, cnt - 1);
                const int rr = e / per, x8 = (e - rr * per) * 8;
                load_row8(X, p, r0 + rr0 + (rr < nr ? rr : nr - 1), x8, o[u]);
              }
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int e = e0 + u * OJA_THREADS;
                if (e >= cnt) break;
                const int rr = e / per, x8 = (e - rr * per) * 8;
                float4* dst = reinterpret_cast<float4*>(Xr + (size_t)rr * d + x8);
                const float z = rr < nr ? 1.f : 0.f;
                dst[0] = make_float4(z * (float)o[u][0], z * (float)o[u][1], z * (float)o[u][2], z * (float)o[u][3]);
                dst[1] = make_float4(z * (float)o[u][4], z * (float)o[u][5], z * (float)o[u][6], z * (float)o[u][7]);
              }
            }
          } else {
            stage16(Xr, (int)(rg * d), [&](int e) {
              const int rr = (int)(e / d);
              const int64_t x = e - (int64_t)rr * d;
              return oja_ld(X, p, r0 + rr0 + (rr < nr ? rr : nr - 1), x);
            });
            for (int e = nr * (int)d + tid; e < rg * (int)d; e += OJA_THREADS) Xr[e] = 0.f;
          }
          __syncthreads();
          staged = rgi;
        }
        if (j < m && !(p.dbg & 256)) {
          float acc[OJA_RG];
#pragma unroll
          for (int rr = 0; rr < OJA_RG; ++rr) acc[rr] = 0.f;
          if (p.wvec) {
            for (int k0 = lane; k0 < n4; k0 += 32 * 8) {
              if (k0 != lane) {
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                  const int k = k0 + 32 * u;
                  w[u] = reinterpret_cast<const float4*>(wj)[k < n4 ? k : n4 - 1];
                }
              }
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                const int k = k0 + 32 * u;
                if (k < n4) {
#pragma unroll
                  for (int rr = 0; rr < OJA_RG; ++rr) {
                    if (rr < rg) {
                      const float4 xv = reinterpret_cast<const float4*>(Xr + (size_t)rr * d)[k];
                      acc[rr] = fmaf(w[u].x, xv.x, acc[rr]);
                      acc[rr] = fmaf(w[u].y, xv.y, acc[rr]);
                      acc[rr] = fmaf(w[u].z, xv.z, acc[rr]);
                      acc[rr] = fmaf(w[u].w, xv.w, acc[rr]);
                    }
                  }
                }
              }
            }
          } else {
            for (int64_t x = lane; x < d; x += 32) {
              const float w = wj[x];
#pragma unroll
              for (int rr = 0; rr < OJA_RG; ++rr)
                if (rr < rg) acc[rr] = fmaf(w, Xr[(size_t)rr * d + x], acc[rr]);
            }
          }
#pragma unroll
          for (int rr = 0; rr < OJA_RG; ++rr) {
            float v = acc[rr];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            acc[rr] = v;
          }
#pragma unroll
          for (int rr = 0; rr < OJA_RG; ++rr)
            if (lane == rr && rr < nr) p.Y[(int64_t)(rr0 + rr) * m + j] = acc[rr];
        }
      }
    }
    if (bclk && st == p.s0) p.clk[4 + blockIdx.x * 3 + 0] = gtimer();
    grid.sync();
    if (rec) p.clk[1] = gtimer();
    // ---- phase 2: Q = X_bᵀY (items of 8 columns) and P = YᵀY (items of 32 4×4 tiles); operands staged
    //      in shared memory as fp64 (Y rows padded to mp), register-blocked, row groups reduced in fixed order
    {
      double* Ys = reinterpret_cast<double*>(smem);                      // [rc][mp]
      double* Xs = Ys + (size_t)rc * mp;                                  // [rc][8]
      double* red = Xs + (size_t)rc * 8;                                  // Q: [gq][mp][8]; P: [32][8][16]
      const int gq = OJA_THREADS / mp;
      for (int it = blockIdx.x; it < ((p.dbg & 32) ? 0 : nq8 + npg); it += gridDim.x) {
        const bool qitem = it < nq8;
        const int64_t xb = qitem ? (int64_t)it * 8 : 0;
        // Q: thread (j, g) over rows g, g+gq, ...;  P: thread (upper tile, g) over rows g, g+32, ...
        const int j = tid % mp, g = tid / mp;
        const int tile = (it - nq8) * 8 + (tid & 7), pg = tid >> 3;
        int ti = 0, tj = tile;
        while (ti < nt4 && tj >= nt4 - ti) {
          tj -= nt4 - ti;
          ++ti;
        }
        tj += ti;
        double acc[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) acc[u] = 0.0;
        for (int rb0 = 0; rb0 < rows; rb0 += rc) {
          const int nr = rows - rb0 < rc ? rows - rb0 : rc;
          const float* ysrc = p.Y + (int64_t)rb0 * m;
          if (p.dbg & 1) {
          } else if (mp == m) {                    // Y rows unpadded: float4 → 2 × double2
            const float4* y4 = reinterpret_cast<const float4*>(ysrc);
            const int n4 = nr * m / 4;
            for (int e0 = tid; e0 < n4; e0 += 8 * OJA_THREADS) {
              float4 v[8];
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                const int e = e0 + u * OJA_THREADS;
                v[u] = y4[e < n4 ? e : n4 - 1];
              }
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                const int e = e0 + u * OJA_THREADS;
                if (e < n4) {
                  double2* o = reinterpret_cast<double2*>(Ys + 4 * e);
                  o[0] = make_double2(v[u].x, v[u].y);
                  o[1] = make_double2(v[u].z, v[u].w);
                }
              }
            }
          } else {
            stage16(Ys, nr * mp, [&](int e) {
              const int r = e / mp, jj = e - r * mp;
              const float v = ysrc[r * m + (jj < m ? jj : m - 1)];
              return jj < m ? (double)v : 0.0;
            });
          }
          if (!qitem || (p.dbg & 1)) {
          } else if (p.xvec && xb + 8 <= d) {      // one row of eight per thread, vector loads
            for (int r = tid; r < nr; r += OJA_THREADS) {
              double o[8];
              load_row8(X, p, r0 + rb0 + r, xb, o);
              double2* dst = reinterpret_cast<double2*>(Xs + r * 8);
#pragma unroll
              for (int u = 0; u < 4; ++u) dst[u] = make_double2(o[2 * u], o[2 * u + 1]);
            }
          } else {
            stage16(Xs, nr * 8, [&](int e) {       // columns past d read column d-1 (their Q is not stored)
              const int64_t x = xb + (e & 7);
              return (double)oja_ld(X, p, r0 + rb0 + (e >> 3), x < d ? x : d - 1);
            });
          }
          __syncthreads();
          if (p.dbg & 2) {
          } else if (qitem) {
            if (g < gq)
              for (int r = g; r < nr; r += gq) {
                const double y = Ys[r * mp + j];
                const double2* xr = reinterpret_cast<const double2*>(Xs + r * 8);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                  const double2 xv = xr[u];
                  acc[2 * u] = fma(y, xv.x, acc[2 * u]);
                  acc[2 * u + 1] = fma(y, xv.y, acc[2 * u + 1]);
                }
              }
          } else if (tile < nup) {
            for (int r = pg; r < nr; r += 32) {
              const double2* yi = reinterpret_cast<const double2*>(Ys + r * mp + ti * 4);
              const double2* yj = reinterpret_cast<const double2*>(Ys + r * mp + tj * 4);
              const double2 i01 = yi[0], i23 = yi[1], j01 = yj[0], j23 = yj[1];
              const double a[4] = {i01.x, i01.y, i23.x, i23.y}, b[4] = {j01.x, j01.y, j23.x, j23.y};
#pragma unroll
              for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[u * 4 + v] = fma(a[u], b[v], acc[u * 4 + v]);
            }
          }
          __syncthreads();
        }
        if (qitem) {
          if (g < gq)
#pragma unroll
            for (int u = 0; u < 8; ++u) red[(g * mp + j) * 8 + u] = acc[u];
          __syncthreads();
          for (int e = tid; e < 8 * m; e += blockDim.x) {
            const int x = e / m, jj = e - x * m;
            double s2 = 0.0;
            for (int gg = 0; gg < gq; ++gg) s2 += red[(gg * mp + jj) * 8 + x];
            if (xb + x < d) p.Q[(xb + x) * m + jj] = s2;
          }
        } else {
#pragma unroll
          for (int u = 0; u < 16; ++u) red[(pg * 8 + (tid & 7)) * 16 + u] = acc[u];
          __syncthreads();
          if (tid < 8 * 16) {
            const int tl = tid >> 4, k = tid & 15;
            int a = 0, b = (it - nq8) * 8 + tl;
            const bool ok = b < nup;
            while (a < nt4 && b >= nt4 - a) {
              b -= nt4 - a;
              ++a;
            }
            b += a;
            const int i = a * 4 + (k >> 2), jj = b * 4 + (k & 3);
            double s2 = 0.0;
            for (int gg = 0; gg < 32; ++gg) s2 += red[(gg * 8 + tl) * 16 + k];
            if (ok && i < m && jj < m) {
              p.P[i * m + jj] = s2;
              p.P[jj * m + i] = s2;
            }
          }
        }
        __syncthreads();
      }
    }
    if (bclk && st == p.s0) p.clk[4 + blockIdx.x * 3 + 1] = gtimer();
    grid.sync();
    if (rec) p.clk[2] = gtimer();
    // the next step's window → L2 while the update runs (phase 1 then stages it from L2, not HBM)
    if (!(p.dbg & 64) && st + 1 < p.s0 + p.steps) {
      const int64_t nblk = (st + 1) % nb;
      const int64_t nrows = nblk < nbf ? p.batch : p.n - nbf * p.batch;
      const size_t row_bytes = (size_t)p.ld * (p.xdtype == PPCA_BF16 ? 2 : 4);
      const char* base = static_cast<const char*>(p.X) + (size_t)(nblk * p.batch) * row_bytes;
      const int64_t lines = (int64_t)((nrows * row_bytes + 127) / 128);
      for (int64_t l = (int64_t)blockIdx.x * OJA_THREADS + tid; l < lines; l += (int64_t)gridDim.x * OJA_THREADS)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(base + l * 128));
    }
    // ---- phase 3: the generalized Oja / Sanger update with Nesterov momentum; item = XC columns, thread
    //      (j, x) with x fastest (W, v coalesced); every load of the item is issued before the first use
    {
      double* Ps = reinterpret_cast<double*>(smem);                      // [m][m]
      float* Ws = reinterpret_cast<float*>(Ps + m * m);                  // [m][xc]: old W[l][xb + xi]
      constexpr int PPT = OJA_MAXM * OJA_MAXM / OJA_THREADS;             // P entries per thread
      const int xi = tid % xc, j = tid / xc;
      bool first = true;
      for (int it = blockIdx.x; it < ((p.dbg & 8) ? 0 : nxc); it += gridDim.x) {
        const int64_t xb = (int64_t)it * xc;
        const int ncol = d - xb < xc ? (int)(d - xb) : xc;
        const bool act = j < m && xi < ncol;
        const int jc = j < m ? j : m - 1;
        const int64_t x = xb + (xi < ncol ? xi : ncol - 1), e = (int64_t)jc * d + x;
        double pv[PPT];
        if (first) {
#pragma unroll
          for (int u = 0; u < PPT; ++u) {
            const int k = tid + u * OJA_THREADS;
            pv[u] = p.P[k < m * m ? k : m * m - 1];
          }
        }
        const float wv = p.W[e];
        const double q = p.Q[x * m + jc];
        const float vo = p.vel[e];
        if (first) {
#pragma unroll
          for (int u = 0; u < PPT; ++u) {
            const int k = tid + u * OJA_THREADS;
            if (k < m * m) Ps[k] = pv[u];
          }
          first = false;
        }
        if (j < m) Ws[j * xc + xi] = wv;
        __syncthreads();
        if (act) {
          const double* pj = Ps + j * m;
          double t0 = 0.0, t1 = 0.0;
          int l = 0;
          for (; l + 1 <= j; l += 2) {
            t0 = fma(pj[l], (double)Ws[l * xc + xi], t0);
            t1 = fma(pj[l + 1], (double)Ws[(l + 1) * xc + xi], t1);
          }
          if (l == j) t0 = fma(pj[l], (double)Ws[l * xc + xi], t0);
          const double g = q - (t0 + t1);
          const double v = p.mu * (double)vo + g;
          const double wn = (double)wv + p.alpha * (g + p.mu * v);
          if (!isfinite(wn)) atomicOr(p.err, DEV_NONFINITE);
          p.vel[e] = (float)v;
          p.W[e] = (float)wn;
        }
        __syncthreads();
      }
    }
    if (bclk && st == p.s0) p.clk[4 + blockIdx.x * 3 + 2] = gtimer();
    grid.sync();
    if (rec) p.clk[3] = gtimer();
  }
}

__global__ void __launch_bounds__(OJA_THREADS, 1) oja_persistent_kernel(OjaParams p) {
  extern __shared__ __align__(16) uint8_t smem[];
  if (p.xdtype == PPCA_F32)
    oja_steps<float>(p, static_cast<const float*>(p.X), smem);
  else if (p.xdtype == PPCA_BF16)
    oja_steps<__nv_bfloat16>(p, static_cast<const __nv_bfloat16*>(p.X), smem);
  else
    oja_steps<SplitF32>(p, static_cast<const SplitF32*>(p.X), smem);
}

// true when the persistent path ran (single GPU, m ≤ 64, automatic pass selection, short windows)
bool oja_persistent(Ctx* c, const ppca_matrix* X, int m, int batch, double alpha, double mu, int64_t s0,
                    int64_t steps, float* W, float* vel, ppca_status* st) {
  *st = PPCA_OK;
  if (c->world != 1 || c->nccl_comm || m > OJA_MAXM || steps <= 0 || c->pass_impl != 0) return false;
  const int64_t d = X->d;
  // short windows only (larger ones run the tensor-core window pass); one staged row must fit
  if ((int64_t)batch * d > ((int64_t)1 << 20) || d * (int64_t)sizeof(float) > OJA_XROW) return false;
  float* Y = (float*)scratch(c, S_Y, (size_t)batch * m * sizeof(float));
  double* Q = (double*)scratch(c, S_PART, (size_t)m * d * sizeof(double) + 8 * (16 + 3 * (size_t)c->sm_count));
  double* P = (double*)scratch(c, S_S, (size_t)m * m * sizeof(double));
  if (!Y || !Q || !P) {
    *st = set_error(c, PPCA_ERR_CUDA, "scratch alloc failed");
    return true;
  }
  static uint64_t attr = 0;
  if (first_on_device(&attr, c->device)) {
    cudaFuncSetAttribute(oja_persistent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, OJA_SMEM);
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, oja_persistent_kernel, OJA_THREADS, OJA_SMEM);
  if (per_sm < 1) return false;
  static const int grid_env = tune_env("PPCA_OJA_GRID", 0);   // experiment builds: fewer CTAs
  const int grid = grid_env > 0 ? std::min(grid_env, c->sm_count) : c->sm_count;
  OjaParams p;
  p.X = X->data; p.xdtype = (int)X->dtype; p.ld = X->ld; p.n = X->n_local; p.d = d;
  p.m = m; p.batch = batch; p.s0 = s0; p.steps = steps;
  p.rg = (int)std::max<int64_t>(1, std::min<int64_t>(OJA_RG, OJA_XROW / (d * (int64_t)sizeof(float))));
  p.xc = std::min(32, OJA_THREADS / m);
  p.rc = std::min(256, (12288 / (((m + 3) & ~3) + 8)) & ~7);
  p.W = W; p.vel = vel; p.Y = Y; p.Q = Q; p.P = P;
  p.alpha = alpha; p.mu = mu; p.err = c->d_err;
  {
    const size_t esz = X->dtype == PPCA_BF16 ? 2 : 4;
    p.xvec = ((uintptr_t)X->data % 16) == 0 && ((size_t)X->ld * esz) % 16 == 0 && d % 8 == 0 ? 1 : 0;
    p.wvec = ((uintptr_t)W % 16) == 0 && d % 4 == 0 ? 1 : 0;
  }
  p.clk = nullptr;
  p.dbg = tune_env("PPCA_OJA_DBG", 0);
  const bool want_clk = tune_env("PPCA_OJA_CLK", 0) != 0;
  if (want_clk) p.clk = (unsigned long long*)(Q + (size_t)m * d);
  void* args[] = {&p};
  cudaError_t e = cudaLaunchCooperativeKernel((void*)oja_persistent_kernel, grid, OJA_THREADS, args, OJA_SMEM,
                                              c->stream);
  if (e == cudaErrorCooperativeLaunchTooLarge) {   // not all CTAs co-resident here (e.g. a shared GPU):
    cudaGetLastError();                               // the per-step launch sequence runs instead
    return false;
  }
  ++c->launches;
  c->last_impl = 1;
  if (e != cudaSuccess) {
    *st = check_cuda(c, e, "oja_persistent_kernel");
    return true;
  }
  if (want_clk) {
    std::vector<unsigned long long> t(4 + 3 * (size_t)grid);
    cudaMemcpyAsync(t.data(), p.clk, t.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream);
    cudaStreamSynchronize(c->stream);
    fprintf(stderr, "[oja_persistent] step phases (ns): Y %llu  Q,P %llu  update %llu  (rg %d xc %d rc %d grid %d)\n",
            t[1] - t[0], t[2] - t[1], t[3] - t[2], p.rg, p.xc, p.rc, grid);
  }
  return true;
}

}  // namespace ppca
