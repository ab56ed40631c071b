// ritz.cuh — single-CTA fp64 Rayleigh–Ritz solve (§8 row a7; Alg. 1 step 4 "full-PCA"):
//   S u = θ B u  with  B = L Lᵀ (Cholesky),  C = L⁻¹ S L⁻ᵀ,  C = U diag(θ) Uᵀ  (parallel cyclic Jacobi),
//   R = Uᵀ L⁻¹  so that the lifted eigenvector i is  e_i = Σ_j R_ij w_j.
// Jacobi uses the round-robin ("circle") pairing: m/2 disjoint rotations per round; A ← JᵀAJ is applied
// block-wise — each (pair, pair) 2×2 block of A transforms independently — so a round costs two
// barriers.  Convergence: off(A) ≤ 1e-12·‖diag A‖_F, at most 100 sweeps.
// Shared memory: A (fp64) and V (fp64 for m ≤ 64, fp32 beyond) plus, for m ≤ 64, L⁻¹ and a temporary.
#pragma once

namespace ritz {

__device__ unsigned long long g_ritz_clk[8];   // phase timestamps of the last ritz_values_kernel (profiling)

__device__ __forceinline__ void pair_of(int r, int i, int mm, int& p, int& q) {
  int a, b;
  if (i == 0) {
    a = 0;
    b = (r % (mm - 1)) + 1;
  } else {
    a = ((i + r) % (mm - 1)) + 1;
    b = ((mm - 1 - i + r) % (mm - 1)) + 1;
  }
  p = a < b ? a : b;
  q = a < b ? b : a;
}

// R == nullptr: eigenvalues only (the per-iterate θ history of power priming) — no V accumulation.
template <typename VT>
__global__ void __launch_bounds__(512) ritz_kernel(const double* __restrict__ S, const double* __restrict__ Bm, int m,
                                                   double* __restrict__ gLinv, double* __restrict__ gT1,
                                                   double* __restrict__ theta, double* __restrict__ R, int* d_err) {
  const bool vectors = R != nullptr;
  extern __shared__ __align__(16) double sm[];
  const int mm = (m + 1) & ~1;          // even (a dummy player for odd m)
  const int np = mm / 2;
  double* A = sm;                                     // mm × mm
  VT* V = reinterpret_cast<VT*>(A + mm * mm);         // mm × mm
  double* tail = reinterpret_cast<double*>(V + mm * mm + (sizeof(VT) == 4 && (mm * mm) % 2 ? 1 : 0));
  const bool small = m <= 64;
  double* Linv = small ? tail : gLinv;                // m × m
  double* T1 = small ? tail + m * m : gT1;            // m × m
  double* misc = small ? tail + 2 * m * m : tail;
  double* diag0 = misc;                               // m
  double* csn = diag0 + mm;                           // 2·np
  int* keep = reinterpret_cast<int*>(csn + 2 * np);   // m
  int* pq = keep + mm;                                // 2·np
  int* perm = pq + 2 * np;                            // m
  __shared__ double red[2][16];
  __shared__ int converged;
  const int tid = threadIdx.x, nt = blockDim.x;

  // 1. L = chol(B) (in A), L⁻¹
  ppca::copy_batched<16>(tid, m * m, nt, [&](int64_t e) { return Bm[e]; }, [&](int64_t e, double v) { A[e] = v; });
  __syncthreads();
  ppca::block_cholesky(A, m, 0.0, keep, diag0, d_err, m);
  ppca::block_lower_inverse(A, m, keep, Linv, m, m);
  // S into A (L is no longer needed), every load in flight at once
  ppca::copy_batched<16>(tid, m * m, nt, [&](int64_t e) { return S[e]; }, [&](int64_t e, double v) { A[e] = v; });
  __syncthreads();
  // 2. C = L⁻¹ S L⁻ᵀ  (T1 = S L⁻ᵀ, then A = L⁻¹ T1), stored mm × mm with a zero dummy row/column
  for (int e = tid; e < m * m; e += nt) {            // lanes vary i: Linv[j][·] is a broadcast
    const int j = e / m, i = e % m;
    double s = 0.0;
    for (int t = 0; t <= j; ++t) s += A[t * m + i] * Linv[j * m + t];   // S symmetric
    T1[i * m + j] = s;
  }
  __syncthreads();
  for (int e = tid; e < mm * mm; e += nt) {
    const int i = e / mm, j = e % mm;
    double s = 0.0;
    if (i < m && j < m)
      for (int t = 0; t <= i; ++t) s += Linv[i * m + t] * T1[t * m + j];
    A[e] = s;
  }
  __syncthreads();
  for (int e = tid; e < mm * mm; e += nt) {
    const int i = e / mm, j = e % mm;
    if (i < j) {
      const double v = 0.5 * (A[i * mm + j] + A[j * mm + i]);
      A[i * mm + j] = v;
      A[j * mm + i] = v;
    }
    if (vectors) V[e] = (VT)(i == j ? 1.0 : 0.0);
  }
  __syncthreads();
  // 3. Jacobi sweeps
  for (int sweep = 0; sweep <= 100; ++sweep) {
    double off = 0.0, dg = 0.0;
    for (int e = tid; e < mm * mm; e += nt) {
      const double v = A[e];
      if (e / mm == e % mm) dg += v * v; else off += v * v;
    }
    off = ppca::warp_sum(off);
    dg = ppca::warp_sum(dg);
    if ((tid & 31) == 0) { red[0][tid >> 5] = off; red[1][tid >> 5] = dg; }
    __syncthreads();
    if (tid == 0) {
      double o = 0, g = 0;
      for (int w = 0; w < nt / 32; ++w) { o += red[0][w]; g += red[1][w]; }
      converged = (sqrt(o) <= 1e-12 * sqrt(g)) || o == 0.0;
      if (!converged && sweep == 100) atomicOr(d_err, ppca::DEV_NOCONV);
    }
    __syncthreads();
    if (converged || sweep == 100) break;
    for (int r = 0; r < mm - 1; ++r) {
      for (int i = tid; i < np; i += nt) {
        int p, q;
        pair_of(r, i, mm, p, q);
        double cc = 1.0, ss = 0.0;
        const double apq = A[p * mm + q];
        if (apq != 0.0) {
          const double tau = (A[q * mm + q] - A[p * mm + p]) / (2.0 * apq);
          const double t = (tau >= 0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
          cc = 1.0 / sqrt(1.0 + t * t);
          ss = t * cc;
        }
        pq[2 * i] = p;
        pq[2 * i + 1] = q;
        csn[2 * i] = cc;
        csn[2 * i + 1] = ss;
      }
      __syncthreads();
      // A ← JᵀAJ one (pair a, pair b) 2×2 block at a time; V ← VJ one (row, pair) couple at a time.
      // Index maps without per-element integer division: thread → (ia, ib) = (tid / np + k·nt/np, tid % np)
      // when np divides nt (m a power of two), else the general e / np map.
      auto block = [&](int ia, int ib) {
        const int p = pq[2 * ia], q = pq[2 * ia + 1], p2 = pq[2 * ib], q2 = pq[2 * ib + 1];
        const double c1 = csn[2 * ia], s1 = csn[2 * ia + 1], c2 = csn[2 * ib], s2 = csn[2 * ib + 1];
        const double a = A[p * mm + p2], b = A[p * mm + q2], c = A[q * mm + p2], d = A[q * mm + q2];
        // rows:  p ← c1·p − s1·q,  q ← s1·p + c1·q ;  columns: p2 ← c2·p2 − s2·q2, q2 ← s2·p2 + c2·q2
        const double ra = c1 * a - s1 * c, rb = c1 * b - s1 * d, rc = s1 * a + c1 * c, rd = s1 * b + c1 * d;
        A[p * mm + p2] = c2 * ra - s2 * rb;
        A[p * mm + q2] = s2 * ra + c2 * rb;
        A[q * mm + p2] = c2 * rc - s2 * rd;
        A[q * mm + q2] = s2 * rc + c2 * rd;
      };
      auto vrot = [&](int ia, int row) {                 // V stored transposed: V[col·mm + row]
        const int p = pq[2 * ia], q = pq[2 * ia + 1];
        const double cc = csn[2 * ia], ss = csn[2 * ia + 1];
        const double vp = (double)V[p * mm + row], vq = (double)V[q * mm + row];
        V[p * mm + row] = (VT)(cc * vp - ss * vq);
        V[q * mm + row] = (VT)(ss * vp + cc * vq);
      };
      if (nt % np == 0) {
        for (int ia = tid / np; ia < np; ia += nt / np) block(ia, tid % np);
      } else {
        for (int e = tid; e < np * np; e += nt) block(e / np, e % np);
      }
      if (vectors) {
        if (nt % mm == 0) {
          for (int ia = tid / mm; ia < np; ia += nt / mm) vrot(ia, tid % mm);
        } else {
          for (int e = tid; e < np * mm; e += nt) vrot(e / mm, e % mm);
        }
      }
      __syncthreads();
    }
  }
  // 4. sort descending (ties by index), R = U_sortedᵀ L⁻¹
  for (int i = tid; i < m; i += nt) {
    const double li = A[i * mm + i];
    int rank = 0;
    for (int j = 0; j < m; ++j) {
      const double lj = A[j * mm + j];
      rank += (lj > li) || (lj == li && j < i);
    }
    perm[rank] = i;
  }
  __syncthreads();
  for (int i = tid; i < m; i += nt) theta[i] = A[perm[i] * mm + perm[i]];
  for (int e = tid; e < (vectors ? m * m : 0); e += nt) {
    const int i = e / m, j = e % m;
    const int col = perm[i];
    double s = 0.0;
    for (int t = j; t < m; ++t) s += (double)V[col * mm + t] * Linv[t * m + j];
    R[e] = s;
  }
}

// Eigenvalues only (the per-iterate θ history of power priming, off the critical path but one per
// iteration): C = L⁻¹SL⁻ᵀ as above, Householder tridiagonalisation of C (4 barriers per column), then all m
// eigenvalues of the tridiagonal by Sturm-count multisection (nt/m threads per eigenvalue, 5 sub-intervals
// per round).  O(m³/nt + m²) instead of Jacobi's O(sweeps·m) barrier rounds.
//
// With R != nullptr (m ≤ 64: the refine) the eigenvectors follow too: one thread per eigenvalue solves the
// twisted factorization of T − θI (top-down LDLᵀ and bottom-up UDUᵀ pivots in shared memory, twist index at
// the smallest |γ_r|, one substitution each way — no iteration); clusters of eigenvalues closer than
// 1e-9·‖T‖ keep inverse iteration (Gaussian elimination with partial pivoting, 3 steps, Gram–Schmidt against
// the cluster's earlier vectors at every step, one thread per cluster); back-transformation by the stored
// Householder reflectors, then R = Uᵀ L⁻¹ in descending order.
__global__ void __launch_bounds__(512) ritz_values_kernel(const double* __restrict__ S, const double* __restrict__ Bm,
                                                          int m, double* __restrict__ gLinv, double* __restrict__ gT1,
                                                          double* __restrict__ theta, int* d_err,
                                                          double* __restrict__ R = nullptr, int top = 0,
                                                          int opt = 0) {
  // top (1 ≤ top ≤ m): only the top largest eigenpairs are formed (the refine needs k of m); 0 = all
  // opt bit 0: Sturm counts by the division-free product recurrence; bit 1: warp-per-row matvec in the
  // tridiagonalisation
  extern __shared__ __align__(16) double sm[];
  if (top <= 0 || top > m) top = m;
  const int jlo = m - top;                            // ascending index of the smallest eigenpair formed
  const bool small = m <= 64;
  const bool vectors = R != nullptr && small;
  double* A = sm;                                     // m × m (C, then the reduced matrix)
  double* Linv = small ? A + m * m : gLinv;
  double* T1 = small ? A + 2 * m * m : gT1;
  __shared__ double diag0[PPCA_MAX_M], vec[PPCA_MAX_M], pv[PPCA_MAX_M], ta[PPCA_MAX_M], tb[PPCA_MAX_M];
  __shared__ double hbeta[PPCA_MAX_M], evals[PPCA_MAX_M];
  __shared__ int keep[PPCA_MAX_M];
  __shared__ double sh_beta;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;

  // 1. L = chol(B), L⁻¹, C = L⁻¹ S L⁻ᵀ (symmetrised)
  if (tid == 0) g_ritz_clk[0] = clock64();
  if (m <= 64 && nt == 512) {                        // register sweep (small.cu): Cholesky and L⁻¹ together
    ppca::chol_inv_sweep2t<2, 16>(Bm, m, Linv, m, d_err, m, keep);
    if (tid == 0) g_ritz_clk[1] = g_ritz_clk[2] = clock64();
  } else {
    ppca::copy_batched<16>(tid, m * m, nt, [&](int64_t e) { return Bm[e]; }, [&](int64_t e, double v) { A[e] = v; });
    __syncthreads();
    ppca::block_cholesky(A, m, 0.0, keep, diag0, d_err, m);
    if (tid == 0) g_ritz_clk[1] = clock64();
    ppca::block_lower_inverse(A, m, keep, Linv, m, m);
    if (tid == 0) g_ritz_clk[2] = clock64();
  }
  ppca::copy_batched<16>(tid, m * m, nt, [&](int64_t e) { return S[e]; }, [&](int64_t e, double v) { A[e] = v; });
  __syncthreads();
  if ((opt & 4) && m == 64 && nt == 512) {
    // both triangular products on 2 × 4 register tiles: OUT[r][c] = Σ_{t ≤ r} L⁻¹[r][t]·B[t][c] with B's rows
    // contiguous along c (16 column tiles per warp: conflict-free 16-byte loads) and two L⁻¹ scalars per t —
    // 4 shared loads per 8 DFMA instead of 2 per 1 (the per-element loops below are bound by shared-memory
    // bandwidth: 25 µs).  Product 1 is (L⁻¹S)ᵀ = S L⁻ᵀ, stored transposed.
    const int tr = tid >> 4, tc = tid & 15, r0 = 2 * tr, c0 = 4 * tc;
    for (int pass = 0; pass < 2; ++pass) {
      const double* Bsrc = pass == 0 ? A : T1;
      double acc[2][4] = {};
      for (int t = 0; t <= r0 + 1; ++t) {
        const double l0 = Linv[r0 * m + t], l1 = Linv[(r0 + 1) * m + t];   // L⁻¹[r0][r0+1] is an exact zero
        const double2 b01 = *reinterpret_cast<const double2*>(Bsrc + t * m + c0);
        const double2 b23 = *reinterpret_cast<const double2*>(Bsrc + t * m + c0 + 2);
        acc[0][0] = fma(l0, b01.x, acc[0][0]);
        acc[0][1] = fma(l0, b01.y, acc[0][1]);
        acc[0][2] = fma(l0, b23.x, acc[0][2]);
        acc[0][3] = fma(l0, b23.y, acc[0][3]);
        acc[1][0] = fma(l1, b01.x, acc[1][0]);
        acc[1][1] = fma(l1, b01.y, acc[1][1]);
        acc[1][2] = fma(l1, b23.x, acc[1][2]);
        acc[1][3] = fma(l1, b23.y, acc[1][3]);
      }
      __syncthreads();                                 // pass 1 overwrites A, which pass 0 read
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          if (pass == 0) T1[(c0 + v) * m + r0 + u] = acc[u][v];   // T1[i][j] = (L⁻¹S)[j][i]
          else A[(r0 + u) * m + c0 + v] = acc[u][v];
        }
      __syncthreads();
    }
  } else {
  for (int e = tid; e < m * m; e += nt) {
    const int j = e / m, i = e % m;
    double s = 0.0;
    for (int t = 0; t <= j; ++t) s += A[t * m + i] * Linv[j * m + t];   // S symmetric (staged in A)
    T1[i * m + j] = s;
  }
  __syncthreads();
  for (int e = tid; e < m * m; e += nt) {
    const int i = e / m, j = e % m;
    double s = 0.0;
    for (int t = 0; t <= i; ++t) s += Linv[i * m + t] * T1[t * m + j];
    A[e] = s;
  }
  __syncthreads();
  }
  for (int e = tid; e < m * m; e += nt) {
    const int i = e / m, j = e % m;
    if (i < j) {
      const double v = 0.5 * (A[i * m + j] + A[j * m + i]);
      A[i * m + j] = v;
      A[j * m + i] = v;
    }
  }
  __syncthreads();
  if (tid == 0) g_ritz_clk[3] = clock64();
  // 2. Householder tridiagonalisation (full symmetric matrix kept up to date), three barriers per column:
  //    (i) warp 0 forms the reflector from row k (= column k: contiguous, no bank conflicts) — norm, α, β, v;
  //    (ii) p = β C'v, each warp also leaving its share of vᵀp; (iii) every thread sums the shares (K = ½β vᵀp)
  //    and applies C' −= v wᵀ + w vᵀ with w = p − K v formed on the fly
  __shared__ double red_k[16];
  for (int k = 0; k + 2 < m; ++k) {
    const int n1 = m - k - 1;
    const double* rowk = A + k * m + (k + 1);          // x_i = A[k][k+1+i] = A[k+1+i][k]
    if (warp == 0) {
      double xs[PPCA_MAX_M / 32], ss = 0.0;
#pragma unroll
      for (int q = 0; q < PPCA_MAX_M / 32; ++q) {
        const int i = lane + 32 * q;
        xs[q] = i < n1 ? rowk[i] : 0.0;
        ss = fma(xs[q], xs[q], ss);
      }
      ss = ppca::warp_sum(ss);
      const double x0 = __shfl_sync(0xffffffffu, xs[0], 0);
      const double alpha = ss > 0.0 ? -copysign(sqrt(ss), x0) : 0.0;
      const double v0 = x0 - alpha;
      const double vtv = ss - x0 * x0 + v0 * v0;
      const double beta = vtv > 0.0 ? 2.0 / vtv : 0.0;
      if (lane == 0) xs[0] = v0;
#pragma unroll
      for (int q = 0; q < PPCA_MAX_M / 32; ++q) {
        const int i = lane + 32 * q;
        if (i < n1) {
          vec[i] = xs[q];
          if (vectors) A[(k + 1 + i) * m + k] = xs[q];   // reflector k kept in column k below the diagonal
        }
      }
      if (lane == 0) {
        sh_beta = beta;
        ta[k] = A[k * m + k];
        tb[k] = alpha;
        if (vectors) hbeta[k] = beta;
      }
    }
    __syncthreads();
    const double beta = sh_beta;
    if (beta != 0.0) {
      // p = β C' v, C' = A[k+1.., k+1..]: G threads per row (consecutive lanes), shuffle-reduced
      const int G = nt / n1 >= 4 ? 4 : (nt / n1 >= 2 ? 2 : 1);
      double vp = 0.0;
      if (opt & 2) {
        // a warp per row, lanes along it (consecutive addresses: no bank conflicts — G lanes per row put the
        // rows of a warp m doubles apart, on the same banks), four rows' reductions interleaved
        const int nw = nt >> 5;
        for (int r0 = warp; r0 < n1; r0 += 4 * nw) {
          double acc[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int i = r0 + u * nw;
            acc[u] = 0.0;
            if (i < n1) {
              const double* row = A + (k + 1 + i) * m + (k + 1);
              for (int j = lane; j < n1; j += 32) acc[u] = fma(row[j], vec[j], acc[u]);
            }
          }
#pragma unroll
          for (int o = 16; o; o >>= 1)
#pragma unroll
            for (int u = 0; u < 4; ++u) acc[u] += __shfl_xor_sync(0xffffffffu, acc[u], o);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int i = r0 + u * nw;
            if (i < n1 && lane == 0) {
              pv[i] = beta * acc[u];
              vp = fma(vec[i], beta * acc[u], vp);
            }
          }
        }
      } else
      for (int b0 = 0; b0 < n1; b0 += nt / G) {
        const int base = b0 + tid / G, q = tid % G;
        const bool act = base < n1;
        double acc = 0.0;
        if (act) {
          const double* row = A + (k + 1 + base) * m + (k + 1);
          for (int j = q; j < n1; j += G) acc = fma(row[j], vec[j], acc);
        }
        for (int o = G / 2; o; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o, G);
        if (act && q == 0) {
          pv[base] = beta * acc;
          vp = fma(vec[base], beta * acc, vp);
        }
      }
      if (!(opt & 2)) vp = ppca::warp_sum(vp);
      if (lane == 0) red_k[warp] = vp;
      __syncthreads();
      double kk = 0.0;
      for (int w2 = 0; w2 < nt / 32; ++w2) kk += red_k[w2];
      const double K = 0.5 * beta * kk;
      // C' −= v wᵀ + w vᵀ,  w = p − K v  (2-D thread map: no integer division per element)
      const int ty = tid >> 5, tx = tid & 31, sy = nt >> 5;
      for (int i = ty; i < n1; i += sy) {
        const double vi = vec[i], wi = pv[i] - K * vi;
        double* Ai = A + (k + 1 + i) * m + (k + 1);
        for (int j = tx; j < n1; j += 32) Ai[j] -= vi * (pv[j] - K * vec[j]) + wi * vec[j];
      }
    }
    __syncthreads();
  }
  if (tid == 0) {
    if (m >= 2) {
      ta[m - 2] = A[(m - 2) * m + (m - 2)];
      tb[m - 2] = A[(m - 1) * m + (m - 2)];
    }
    ta[m - 1] = A[(m - 1) * m + (m - 1)];
  }
  __syncthreads();
  if (tid == 0) g_ritz_clk[4] = clock64();
  // 3. Sturm multisection: eigenvalue j (ascending) by G = nt/top threads; count(x) = #{i : d_i < 0}
  double lo = 0.0, hi = 0.0;
  for (int i = 0; i < m; ++i) {                        // Gershgorin bounds (every thread)
    const double r = (i > 0 ? fabs(tb[i - 1]) : 0.0) + (i + 1 < m ? fabs(tb[i]) : 0.0);
    lo = i == 0 ? ta[i] - r : fmin(lo, ta[i] - r);
    hi = i == 0 ? ta[i] + r : fmax(hi, ta[i] + r);
  }
  const double span = fmax(hi - lo, 1e-300);
  lo -= 1e-12 * span;
  hi += 1e-12 * span;
  // θ history needs ~1e-10 relative (the parity bar is 1e-4): (G+1)^rounds ≥ 2^42 of the Gershgorin span.
  // (The Sturm recurrence is bound by the fp64 reciprocal's throughput, not its latency: four interleaved
  // probes per thread and 9 rounds of 32 probes measured 215 µs against 94 µs for 14 rounds of 8.)
  // (16 probes × 11 rounds for top = 32 measured 84 µs against 81 µs for 8 × 14: the counts share the fp64
  // reciprocal pipe, so more probes per round do not pay)
  const int G = nt / top >= 8 ? 8 : (nt / top >= 4 ? 4 : (nt / top >= 2 ? 2 : 1));
  const int rounds = G == 8 ? 14 : (G == 4 ? 19 : (G == 2 ? 27 : 42));
  // squared off-diagonal once (bsq[i] = b_{i-1}², bsq[0] unused), so the count loop is load + rcp + two DFMA
  double* bsq = pv;                                   // (pv is free after the tridiagonalisation)
  double* tas = vec;                                  // a_i / span (vec is free too)
  const double inv_span = 1.0 / span;
  for (int i = tid; i < m; i += nt) {
    const double bi = i > 0 ? tb[i - 1] : 0.0;
    if (opt & 1) {
      const double bs = bi * inv_span;
      bsq[i] = bs * bs;
      tas[i] = ta[i] * inv_span;
    } else {
      bsq[i] = bi * bi;
    }
  }
  __syncthreads();
  for (int b0 = jlo; b0 < m; b0 += nt / G) {            // uniform trip counts: every lane reaches the shuffles
    const int q = tid % G, j = b0 + tid / G;
    const bool act = j < m;
    const int mm = act ? m : 0;
    double L = lo, U = hi;
    for (int round = 0; round < rounds; ++round) {
      const double x = L + (U - L) * (double)(q + 1) / (double)(G + 1);
      int cnt = 0;
      if (opt & 1) {
        // Sturm count without the reciprocal: q_{i+1} = (a_i − x)·q_i − b_{i−1}²·q_{i−1} (q_0 = 1), the leading
        // principal minors of T − xI, d_i = q_{i+1}/q_i; count = sign changes along q.  One dependent DFMA per
        // row instead of reciprocal + DFMA.  T is scaled by 1/span (|a − x| ≤ 1, b² ≤ 1: growth ≤ 2 per row, no
        // overflow in 128 rows); the pair is rescaled by a power of two every second row against underflow; an
        // exact zero takes the sign opposite to its predecessor (the d_i = −tiny rule of the quotient form).
        const double xs = x * inv_span;
        double qp = 1.0, qc = tas[0] - xs;
        if (qc == 0.0) qc = -1e-280;
        cnt += qc < 0.0;
#pragma unroll 2
        for (int i = 1; i < mm; ++i) {
          double qn = fma(tas[i] - xs, qc, -(bsq[i] * qp));
          if (qn == 0.0) qn = -copysign(1e-280, qc);
          cnt += ((__double2hiint(qn) ^ __double2hiint(qc)) >> 31) & 1;
          qp = qc;
          qc = qn;
          if (i & 1) {                                 // 2^−e, e the exponent of max(|q_i|, |q_{i+1}|)
            const int eh = __double2hiint(fmax(fabs(qc), fabs(qp))) & 0x7ff00000;
            const double sc = __hiloint2double(0x7fe00000 - eh, 0);
            qc *= sc;
            qp *= sc;
          }
        }
      } else {
        double dd = ta[0] - x;
        if (dd == 0.0) dd = -1e-300;
        cnt += dd < 0.0;
#pragma unroll 4
        for (int i = 1; i < mm; ++i) {                 // (reciprocal instead of an IEEE division: only signs count)
          dd = (ta[i] - x) - bsq[i] * __drcp_rn(dd);
          if (dd == 0.0) dd = -1e-300;
          cnt += dd < 0.0;
        }
      }
      if (!act) cnt = 0;
      // the G probes split [L, U] into G+1 parts: keep the part holding the (j+1)-th eigenvalue
      double nL = L, nU = U;
      for (int g2 = 0; g2 < G; ++g2) {
        const int c2 = __shfl_sync(0xffffffffu, cnt, (lane & ~(G - 1)) + g2, 32);
        const double x2 = L + (U - L) * (double)(g2 + 1) / (double)(G + 1);
        if (c2 <= j) nL = x2;
        else if (x2 < nU) nU = x2;
      }
      L = nL;
      U = nU;
    }
    if (act && q == 0) {
      theta[m - 1 - j] = 0.5 * (L + U);                // descending
      evals[j] = 0.5 * (L + U);
    }
  }
  __syncthreads();
  if (tid == 0) g_ritz_clk[5] = clock64();
  if (!vectors) return;
  // 4. eigenvectors of T: inverse iteration, one thread per cluster of close eigenvalues
  double* XT = T1;                                    // XT[i·m + j] = component i of eigenvector j (ascending)
  // clusters: gaps ≤ 1e-9·‖T‖.  Inverse iteration separates eigenvalues whose gap δ exceeds the shifts'
  // error (~ε‖T‖) and leaves the vectors orthogonal to ~ε‖T‖/δ ≤ 2e-7 here (below the fp32 outputs'
  // rounding); LAPACK's 1e-3·‖T‖ would put most of a power-law spectrum (C4: gaps 1.5·j^-2.5·λ₁) into
  // one serial Gram–Schmidt chain (8.5 ms per refine, measured)
  const double ctol = 1e-9 * fmax(fabs(lo), fabs(hi));
  const double tiny = 1e-14 * span;
  double* Dp = A + 3 * m * m;                         // Dp[i·m + j], Dm[i·m + j]: pivots of eigenvalue j's twist
  double* Dm = A + 4 * m * m;
  for (int j0 = jlo + tid; j0 < m; j0 += nt) {
    if (j0 > jlo && evals[j0] - evals[j0 - 1] <= ctol) continue;   // not a cluster leader
    int j1 = j0 + 1;
    while (j1 < m && evals[j1] - evals[j1 - 1] <= ctol) ++j1;
    if (j1 == j0 + 1) {
      // isolated eigenvalue: twisted factorization  T − σI = L₊D₊L₊ᵀ = U₋D₋U₋ᵀ,  γ_r = D₊_r + D₋_r − (a_r − σ);
      // z_r = 1, z_i = −(b_i / D₊_i)·z_{i+1} above r, z_i = −(b_{i−1} / D₋_i)·z_{i−1} below r
      const int j = j0;
      const double sg = evals[j];
      auto guard = [&](double v) { return fabs(v) < tiny ? (v < 0.0 ? -tiny : tiny) : v; };
      double dp = guard(ta[0] - sg);
      Dp[j] = dp;
      for (int i = 1; i < m; ++i) {
        dp = guard((ta[i] - sg) - tb[i - 1] * (tb[i - 1] / dp));
        Dp[i * m + j] = dp;
      }
      double dm = guard(ta[m - 1] - sg);
      Dm[(m - 1) * m + j] = dm;
      for (int i = m - 2; i >= 0; --i) {
        dm = guard((ta[i] - sg) - tb[i] * (tb[i] / dm));
        Dm[i * m + j] = dm;
      }
      int r = 0;
      double gbest = 1e300;
      for (int i = 0; i < m; ++i) {
        const double g = fabs(Dp[i * m + j] + Dm[i * m + j] - (ta[i] - sg));
        if (g < gbest) { gbest = g; r = i; }
      }
      double z = 1.0, nn = 1.0;
      XT[r * m + j] = 1.0;
      for (int i = r - 1; i >= 0; --i) {
        z = -(tb[i] / Dp[i * m + j]) * z;
        XT[i * m + j] = z;
        nn = fma(z, z, nn);
      }
      z = 1.0;
      for (int i = r + 1; i < m; ++i) {
        z = -(tb[i - 1] / Dm[i * m + j]) * z;
        XT[i * m + j] = z;
        nn = fma(z, z, nn);
      }
      const double rn = rsqrt(nn);
      for (int i = 0; i < m; ++i) XT[i * m + j] *= rn;
      continue;
    }
    for (int j = j0; j < j1; ++j) {
      double dl[PPCA_MAX_M / 2], d[PPCA_MAX_M / 2], du[PPCA_MAX_M / 2], du2[PPCA_MAX_M / 2], x[PPCA_MAX_M / 2];
      bool sw[PPCA_MAX_M / 2];
      const double sg = evals[j];
      for (int i = 0; i < m; ++i) {
        d[i] = ta[i] - sg;
        if (i + 1 < m) { du[i] = tb[i]; dl[i] = tb[i]; }
        du2[i] = 0.0;
        sw[i] = false;
      }
      for (int i = 0; i + 1 < m; ++i) {              // tridiagonal LU with partial pivoting
        if (fabs(d[i]) >= fabs(dl[i])) {
          if (d[i] == 0.0) d[i] = tiny;
          const double f = dl[i] / d[i];
          dl[i] = f;
          d[i + 1] -= f * du[i];
        } else {
          const double f = d[i] / dl[i];
          d[i] = dl[i];
          dl[i] = f;
          const double t = du[i];
          du[i] = d[i + 1];
          d[i + 1] = t - f * d[i + 1];
          if (i + 2 < m) {
            du2[i] = du[i + 1];
            du[i + 1] = -f * du[i + 1];
          }
          sw[i] = true;
        }
      }
      if (fabs(d[m - 1]) < tiny) d[m - 1] = d[m - 1] < 0.0 ? -tiny : tiny;
      // U's diagonal as reciprocals once (the solves below then multiply: 3·m fp64 divisions saved)
      for (int i = 0; i < m; ++i) d[i] = 1.0 / (fabs(d[i]) < tiny ? (d[i] < 0.0 ? -tiny : tiny) : d[i]);
      for (int i = 0; i < m; ++i) x[i] = 1.0 + 0.37 * sin(0.9 * (double)(i + 1) * (double)(j + 1));
      for (int it = 0; it < 3; ++it) {
        for (int i = 0; i + 1 < m; ++i) {              // L
          if (!sw[i]) {
            x[i + 1] -= dl[i] * x[i];
          } else {
            const double t = x[i];
            x[i] = x[i + 1];
            x[i + 1] = t - dl[i] * x[i];
          }
        }
        x[m - 1] *= d[m - 1];                          // U (d holds 1/U_ii)
        if (m >= 2) x[m - 2] = (x[m - 2] - du[m - 2] * x[m - 1]) * d[m - 2];
        for (int i = m - 3; i >= 0; --i) x[i] = (x[i] - du[i] * x[i + 1] - du2[i] * x[i + 2]) * d[i];
        for (int jp = j0; jp < j; ++jp) {              // Gram–Schmidt against the cluster's earlier vectors
          double dt = 0.0;
          for (int i = 0; i < m; ++i) dt += XT[i * m + jp] * x[i];
          for (int i = 0; i < m; ++i) x[i] -= dt * XT[i * m + jp];
        }
        double nn = 0.0;
        for (int i = 0; i < m; ++i) nn += x[i] * x[i];
        const double rn = nn > 0.0 ? rsqrt(nn) : 0.0;
        for (int i = 0; i < m; ++i) x[i] *= rn;
      }
      for (int i = 0; i < m; ++i) XT[i * m + j] = x[i];
    }
  }
  __syncthreads();
  if (tid == 0) g_ritz_clk[6] = clock64();
  // 5. back-transformation y = H_0 ⋯ H_{m-3} x.  Thread (j, s): lane-consecutive vectors j (conflict-free
  //    XT columns, reflector entries broadcast), s = one of nt/64 row slices; per reflector the slices'
  //    partial dot products meet in shared memory (two barriers per reflector)
  {
    const int ns = nt / 64 < 1 ? 1 : (nt / 64 > 8 ? 8 : nt / 64);
    const int j = tid % 64, sl = tid / 64;
    const bool own = j >= jlo && j < m && sl < ns;
    __shared__ double red[8 * 64];                    // ns × 64 partial dots
    for (int k = m - 3; k >= 0; --k) {
      const double bk = hbeta[k];
      if (bk == 0.0) continue;
      const int n1 = m - k - 1;
      double dt = 0.0;
      if (own)
        for (int i = sl; i < n1; i += ns) dt += A[(k + 1 + i) * m + k] * XT[(k + 1 + i) * m + j];
      if (own) red[sl * 64 + j] = dt;
      __syncthreads();
      if (own) {
        double tot = 0.0;
        for (int q = 0; q < ns; ++q) tot += red[q * 64 + j];
        tot *= bk;
        for (int i = sl; i < n1; i += ns) XT[(k + 1 + i) * m + j] -= tot * A[(k + 1 + i) * m + k];
      }
      __syncthreads();
    }
  }
  if (tid == 0) g_ritz_clk[7] = clock64();
  // 6. R = Uᵀ L⁻¹ in descending order (row i ↔ ascending eigenvector m-1-i)
  for (int e = tid; e < top * m; e += nt) {
    const int i = e / m, c = e % m;
    const int j = m - 1 - i;
    double sum = 0.0;
    for (int t = c; t < m; ++t) sum += XT[t * m + j] * Linv[t * m + c];
    R[e] = sum;
  }
}

inline size_t values_smem_bytes(int m) { return (size_t)(m <= 64 ? 3 : 1) * m * m * sizeof(double); }
// with eigenvectors (m ≤ 64): + the twisted factorizations' pivots (2 · m × m)
inline size_t vectors_smem_bytes(int m) { return (size_t)5 * m * m * sizeof(double); }

inline size_t smem_bytes(int m) {
  const int mm = (m + 1) & ~1;
  const bool small = m <= 64;
  size_t b = (size_t)mm * mm * 8 + (size_t)mm * mm * (small ? 8 : 4) + 8;
  if (small) b += (size_t)2 * m * m * 8;
  b += (size_t)mm * 8 + (size_t)mm * 8 + (size_t)mm * 4 + (size_t)mm * 4 + (size_t)mm * 4 + 64;
  return b;
}

}  // namespace ritz
