"""Full-size checks (BASELINE.json configs[2] = C3 and configs[4] = C5) in the launch configuration bench.py
times: the split / bf16 X on one GPU, the tcgen05 pass, power priming with per-iterate Ritz values, refine.

The fp64 oracle cannot stream these sizes in seconds, so the checks are (i) outputs it can compute one by
one — generator rows sampled across the shard, including the ragged last tile — and (ii) properties that
hold at any size (Alg. 1 L47-51; readings R23):
  * Cauchy interlacing of the pPCA Ritz values with the spectrum of XᵀX (C3: d = 1024, from the library's
    fp64 Gram), identity of pPCA on exact eigenvectors;
  * idempotence (refine of its own output), captured variance of each Ritz vector = its Ritz value;
  * θ₁ of block power non-decreasing over iterations; Ky Fan sums of pPCA ≥ those of the priming vectors;
  * agreement of two independent kernels (tcgen05 split-bf16 pass vs exact-fp32 CUDA-core pass) within the
    north-star tolerances (Ritz 1e-4 relative, 1e-3 for the bf16-stored C5).
"""
import math

import numpy as np
import pytest

from inputs import configs as C
from inputs import generate as G
from tests import gpu_util as U

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def P():
    import paper_2109_03709_b200 as P
    P.load()
    return P


@pytest.fixture(scope="module")
def ctx(P):
    import torch
    torch.cuda.init()
    h = P.ppca_ctx_create(0, torch.cuda.current_stream())
    yield h
    P.ppca_ctx_destroy(h)


def _sample_rows(n):
    rng = np.random.default_rng(42)
    return np.unique(np.concatenate([[0, 1, 127, 128, n - 129, n - 2, n - 1], rng.integers(0, n, 9)]))


def _gen(P, ctx, w, split):
    import torch
    s = w.spec
    dt = torch.float32 if s.dtype == "f32" else torch.bfloat16
    X = torch.empty((s.n, s.d), dtype=dt, device="cuda")
    _, mu = P.ppca_generate(ctx, P.gen_spec(s), X)
    return X, mu


def _check_rows(X, mu, spec):
    """Sampled stored rows (+ the reported mean) against the host generator's raw rows."""
    import torch
    rows = _sample_rows(spec.n)
    raw = G.raw_rows(spec, rows)
    if spec.dtype == "f32":
        got = X[torch.from_numpy(rows).cuda()].double().cpu().numpy()
        tol = np.spacing(np.abs(got).astype(np.float32)).astype(np.float64) + 1e-12 * np.abs(mu)
    else:
        got = X[torch.from_numpy(rows).cuda()].float().double().cpu().numpy()
        tol = np.abs(got) * 2.0 ** -8 + 1e-30
    np.testing.assert_array_less(np.abs(got + mu[None, :] - raw), tol + 1e-9 * np.abs(raw) + 1e-12)


def _power_and_refine(P, ctx, Xm, w, iters, impl, d):
    import torch
    P.ppca_set_pass_impl(ctx, impl)
    try:
        W = torch.zeros((w.m, d), dtype=torch.float32, device="cuda")
        th_hist = P.ppca_prime_power(ctx, Xm, w.m, iters, w.init_seed, W, theta_hist=True)
        E = torch.zeros((w.k, d), dtype=torch.float32, device="cuda")
        th, dim = P.ppca_refine(ctx, Xm, W, w.m, w.k, E)
        used = P.ppca_last_pass_impl(ctx)
    finally:
        P.ppca_set_pass_impl(ctx, 0)
    return W, th_hist, E, th, dim, used


def _properties(P, ctx, Xm, w, W, th_hist, E, th, tol):
    import torch
    # θ₁ of block power never decreases (Rayleigh quotient of the dominant direction, P L61-63)
    t1 = th_hist[:, 0]
    assert np.all(np.diff(t1) >= -tol * t1[1:]), t1
    # idempotence of pPCA (Alg. 1 applied to its own output)
    E2 = torch.zeros_like(E)
    th2, _ = P.ppca_refine(ctx, Xm, E, w.k, w.k, E2)
    assert U.ritz_rel_err(th2, th) < tol
    cos = U.abs_cos(E2.cpu().numpy(), E.cpu().numpy())
    gi = U.gapped(th, w.k)
    assert cos[gi].min() > 0.9999
    # captured variance ‖Xe_i‖² of each Ritz vector equals its Ritz value (P L416)
    var = P.ppca_captured_variance(ctx, Xm, E, w.k)
    np.testing.assert_allclose(var, th, rtol=tol)
    # Ky Fan (R23): Σ_{i≤j} θ_i ≥ Σ_{i≤j} ρ_(i) of the (orthonormal) priming vectors
    rho = np.sort(P.ppca_captured_variance(ctx, Xm, W, w.m))[::-1]
    _, thm = th, th
    assert th[0] >= rho[0] * (1 - tol)
    for j in range(w.k):
        assert th[: j + 1].sum() >= rho[: j + 1].sum() * (1 - tol)


def test_c3_full_size(P, ctx):
    """C3 (n = 10⁶, d = 1024, fp32 stored as split planes, m = 64): generator rows, interlacing with the
    exact spectrum, pPCA identity on eigenvectors, properties, tcgen05 vs CUDA-core pass."""
    import torch
    w = C.C3
    s = w.spec
    X, mu = _gen(P, ctx, w, split=False)
    _check_rows(X, mu, s)
    # exact spectrum of XᵀX (fp64 Gram over all rows) for interlacing / identity
    Xm32 = P.matrix(X)
    G64 = torch.zeros((s.d, s.d), dtype=torch.float64, device="cuda")
    P.ppca_gram(ctx, Xm32, G64)
    lam, V = np.linalg.eigh(G64.cpu().numpy())
    lam, T = lam[::-1], V[:, ::-1].T.copy()
    iters = 5
    # reference kernel: exact-fp32 CUDA-core pass on the plain fp32 X
    W1, h1, E1, th1, _, used1 = _power_and_refine(P, ctx, Xm32, w, iters, 1, s.d)
    assert used1 == 1
    # bench path: split planes, tcgen05
    P.ppca_split_f32(ctx, X, s.d)
    Xm = P.matrix(X, split=True)
    W2, h2, E2, th2, dim, used2 = _power_and_refine(P, ctx, Xm, w, iters, 2, s.d)
    assert used2 == 2 and dim == w.m
    tol = 1e-4
    for t in range(iters):
        assert U.ritz_rel_err(h2[t], h1[t]) < tol, f"iteration {t}"
    assert U.ritz_rel_err(th2, th1) < tol
    gi = U.gapped(th1, w.k)
    cos = U.abs_cos(E2.cpu().numpy(), E1.cpu().numpy())
    assert cos[gi].min() >= 0.9999
    # Cauchy interlacing λ_{i+d−m} ≤ θ_i ≤ λ_i (P L260-269: restriction of XᵀX to span W)
    d, m = s.d, w.m
    for i in range(w.k):
        assert lam[i + d - m] * (1 - tol) <= th2[i] <= lam[i] * (1 + tol)
    # after 5 iterations the C3 pPCA vectors reach LCES = k at π/1024 (bench time-to-LCES)
    lc, _ = U.lces_all(E2.cpu().numpy(), T[: w.k])
    assert lc[-1] == w.k, lc
    # pPCA is the identity on exact eigenvectors (l = 0)
    Tt = torch.from_numpy(T[: w.k].astype(np.float32)).cuda()
    E3 = torch.zeros_like(Tt)
    th3, _ = P.ppca_refine(ctx, Xm, Tt, w.k, w.k, E3)
    np.testing.assert_allclose(th3, lam[: w.k], rtol=tol)
    assert U.abs_cos(E3.cpu().numpy(), T[: w.k]).min() > 0.9999
    _properties(P, ctx, Xm, w, W2, h2, E2, th2, tol)


def test_c5_full_size(P, ctx):
    """C5 (n = 2·10⁵, d = 65536, bf16, m = 128): generator rows, properties, tcgen05 vs CUDA-core pass."""
    w = C.C5
    s = w.spec
    X, mu = _gen(P, ctx, w, split=False)
    _check_rows(X, mu, s)
    Xm = P.matrix(X)
    iters = 3
    W1, h1, E1, th1, _, used1 = _power_and_refine(P, ctx, Xm, w, iters, 1, s.d)
    W2, h2, E2, th2, dim, used2 = _power_and_refine(P, ctx, Xm, w, iters, 2, s.d)
    assert used1 == 1 and used2 == 2 and dim == w.m
    tol = 1e-3
    for t in range(iters):
        assert U.ritz_rel_err(h2[t], h1[t]) < tol, f"iteration {t}"
    assert U.ritz_rel_err(th2, th1) < tol
    _properties(P, ctx, Xm, w, W2, h2, E2, th2, tol)
