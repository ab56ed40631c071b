"""Full-size checks of BASELINE.json configs[1..4] (C2, C3, C4, C5) in the launch configuration bench.py
times: the split / bf16 X on one GPU, the tcgen05 pass, power priming with per-iterate Ritz values,
minibatch primings, refine.  C2 (60000 x 784) is small enough for the fp64 oracle itself.

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


def test_c3_full_size_power_and_refine_vs_oracle(P, ctx):
    """C3 (BASELINE configs[2]) at its full size, 10⁶ x 1024, against the fp64 oracle directly, in the bench's
    launch configuration: the split layout, the d-sliced pair kernel (73–74 clusters over 1e6 rows), 4 block
    power iterations from the seeded start (the time-to-LCES count) and the refine — per-iterate Ritz values
    1e-4, the primed subspace, refine Ritz values / |cos| where gapped, identical LCES at all thresholds.
    The oracle streams the stored X (the device generator's output, itself checked against the host
    generator on sampled rows in test_c3_full_size) in fp64: ~8 GB of host memory, ~1 TFLOP of numpy."""
    import torch
    from oracle import ppca_oracle as O
    w = C.C3
    s = w.spec
    iters = 4
    X, mu = _gen(P, ctx, w, split=False)
    X64 = X.cpu().numpy().astype(np.float64)
    P.ppca_split_f32(ctx, X, s.d)
    Xm = P.matrix(X, split=True)
    W0 = G.init_gaussians(w.init_seed, w.m, s.d)
    W_ref, S_hist = O.prime_power(X64, W0, iters)
    E_ref, th_ref, th_all_ref, _ = O.ppca_refine(X64, W_ref, w.k)
    G64 = X64.T @ X64
    lam, V = np.linalg.eigh(G64)
    T = O.sign_convention(V[:, ::-1][:, : w.k].T.copy())
    del G64, X64
    W = torch.zeros((w.m, s.d), dtype=torch.float32, device="cuda")
    P.ppca_set_pass_impl(ctx, 0)
    hist = P.ppca_prime_power(ctx, Xm, w.m, iters, w.init_seed, W, theta_hist=True)
    assert P.ppca_last_power_kernel(ctx) == 4, "expected the d-sliced pair kernel (the bench's configuration)"
    worst = 0.0
    for t in range(iters):
        e = U.ritz_rel_err(hist[t], O.ritz_values(S_hist[t]))
        worst = max(worst, e)
        assert e < 1e-4, f"C3 full iteration {t}: {e:.3e}"
    Wh = W.cpu().numpy().astype(np.float64)
    assert np.linalg.svd(Wh @ W_ref.T, compute_uv=False).min() > 1 - 1e-4
    E = torch.zeros((w.k, s.d), dtype=torch.float32, device="cuda")
    th, dim = P.ppca_refine(ctx, Xm, W, w.m, w.k, E)
    assert dim == w.m
    err = U.assert_ppca_parity(E.cpu().numpy(), th, E_ref, th_ref, T, 1e-4, "C3 full", th_all_ref)
    lc, _ = U.lces_all(E.cpu().numpy(), T)
    lc_ref, _ = U.lces_all(E_ref, T)
    assert lc == lc_ref, f"LCES {lc} vs oracle {lc_ref}"
    print(f"\n[parity] C3 full: per-iterate Ritz err {worst:.2e}, refine {err:.3e}, LCES {lc}")


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


def test_c2_full_size_oja_against_oracle(P, ctx):
    """C2 (BASELINE configs[1]) at its full size, 60000 x 784, against the fp64 oracle directly: the whole
    stored X, 10 epochs (2350 steps) of generalized Oja (b = 256, α = 1e-3, Nesterov 0.9; readings R8-R10),
    the pPCA refine (Ritz values 1e-4, |cos| where gapped, identical LCES)."""
    import torch
    from oracle import ppca_oracle as O
    w = C.C2
    s = w.spec
    Xs = G.dataset(s)
    X64 = G.stored_to_f64(Xs, s.dtype)
    lam, T = O.truth(X64)
    steps = 2350
    W_ref, _ = O.prime_oja(X64, G.init_gaussians(w.init_seed, w.m, s.d), w.batch, w.alpha, w.momentum, steps)
    E_ref, th_ref, th_all_ref, _ = O.ppca_refine(X64, W_ref, w.k)
    X = torch.empty((s.n, s.d), dtype=torch.float32, device="cuda")
    P.ppca_generate(ctx, P.gen_spec(s), X)
    np.testing.assert_array_less(np.abs(X.cpu().numpy() - Xs), np.spacing(np.abs(Xs)) * 1.01 + 1e-30)
    P.ppca_split_f32(ctx, X, s.d)
    Xm = P.matrix(X, split=True)
    W = torch.zeros((w.m, s.d), dtype=torch.float32, device="cuda")
    vel = torch.zeros_like(W)
    assert P.ppca_prime_oja(ctx, Xm, w.m, w.batch, w.alpha, w.momentum, steps, w.init_seed, W, vel, 0) == steps
    rel = np.linalg.norm(W.cpu().numpy() - W_ref) / np.linalg.norm(W_ref)
    assert rel < 1e-3, f"Oja trajectory drift {rel:.2e}"
    E = torch.zeros((w.k, s.d), dtype=torch.float32, device="cuda")
    th, _ = P.ppca_refine(ctx, Xm, W, w.m, w.k, E)
    err = U.assert_ppca_parity(E.cpu().numpy(), th, E_ref, th_ref, T, 1e-4, "C2 full", th_all_ref)
    lc, _ = U.lces_all(E.cpu().numpy(), T[: w.k])
    print(f"\n[parity] C2 full: Oja drift {rel:.2e}, Ritz rel err {err:.3e}, LCES {lc}")


def test_c4_full_size_eigengame_properties(P, ctx):
    """C4 (BASELINE configs[3]) at its full size, 2·10⁶ x 4096 fp32 (split layout, 32.8 GB): EigenGame steps
    on the tensor-core window pass against the exact-fp32 CUDA-core pass from the same start, then the
    refine's properties (idempotence, captured variance = θ, Ky Fan) and Cauchy interlacing with the exact
    spectrum of XᵀX (fp64 Gram over all rows)."""
    import torch
    w = C.C4
    s = w.spec
    X = torch.empty((s.n, s.d), dtype=torch.float32, device="cuda")
    _, mu = P.ppca_generate(ctx, P.gen_spec(s), X)
    _check_rows(X, mu, s)
    G64 = torch.zeros((s.d, s.d), dtype=torch.float64, device="cuda")
    P.ppca_gram(ctx, P.matrix(X), G64)
    lam = np.linalg.eigvalsh(G64.cpu().numpy())[::-1]
    del G64
    P.ppca_split_f32(ctx, X, s.d)
    Xm = P.matrix(X, split=True)
    steps = 20
    out = {}
    for impl in (1, 2):
        P.ppca_set_pass_impl(ctx, impl)
        try:
            V = torch.zeros((w.m, s.d), dtype=torch.float32, device="cuda")
            vel = torch.zeros_like(V)
            P.ppca_prime_eigengame(ctx, Xm, w.m, w.batch, w.alpha, w.momentum, steps, w.init_seed, V, vel, 0)
            out[impl] = (V.clone(), P.ppca_last_pass_impl(ctx))
        finally:
            P.ppca_set_pass_impl(ctx, 0)
    assert out[1][1] == 1 and out[2][1] == 2
    V1, V2 = out[1][0].cpu().numpy().astype(np.float64), out[2][0].cpu().numpy().astype(np.float64)
    rel = np.linalg.norm(V2 - V1) / np.linalg.norm(V1)
    assert rel < 1e-3, f"tensor-core vs CUDA-core EigenGame trajectories differ by {rel:.2e}"
    E = torch.zeros((w.k, s.d), dtype=torch.float32, device="cuda")
    V = out[2][0]
    th, dim = P.ppca_refine(ctx, Xm, V, w.m, w.k, E)
    assert dim == w.m
    tol = 1e-4
    d, m = s.d, w.m
    for i in range(w.k):
        assert lam[i + d - m] * (1 - tol) <= th[i] <= lam[i] * (1 + tol)
    E2 = torch.zeros_like(E)
    th2, _ = P.ppca_refine(ctx, Xm, E, w.k, w.k, E2)
    assert U.ritz_rel_err(th2, th) < tol
    var = P.ppca_captured_variance(ctx, Xm, E, w.k)
    np.testing.assert_allclose(var, th, rtol=tol)
    print(f"\n[parity] C4 full: EigenGame TC vs SIMT drift {rel:.2e}, theta_1/lambda_1 {th[0] / lam[0]:.6f}")
