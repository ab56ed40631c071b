"""GPU (C-ABI) vs fp64 oracle on the same seeded inputs — the parity gate.

Sizes are the reduced workloads of inputs/configs.SMALL (several row tiles and a ragged
tail).  Tolerances are BASELINE.json north_star's: Ritz values 1e-4 relative (1e-3 for the
bf16-stored config), |cos| ≥ 0.9999 where the relative eigengap > 1e-2, identical LCES.
"""
import math

import numpy as np
import pytest

from inputs import configs as C
from inputs import generate as G
from oracle import ppca_oracle as O
from tests import gpu_util as U

pytestmark = pytest.mark.gpu


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


def _tol(spec):
    return 1e-3 if spec.dtype == "bf16" else 1e-4


def _host(w):
    Xs = G.dataset(w.spec)
    return Xs, G.stored_to_f64(Xs, w.spec.dtype)


# ----------------------------------------------------------------------------- generator
def test_philox_words_match_host_and_kat(P, ctx):
    import torch
    from inputs import philox as ph
    out = torch.zeros(4, dtype=torch.int32, device="cuda")
    P.ppca_philox_words(ctx, 0, 0, 0, out)
    assert [int(x) & 0xFFFFFFFF for x in out.cpu()] == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    for seed, stream, first, cnt in [(1002, 0, 0, 1000), (2**40 + 7, 5, 12345, 333), (9, 1, 2**33 + 1, 64)]:
        out = torch.zeros(cnt, dtype=torch.int32, device="cuda")
        P.ppca_philox_words(ctx, seed, stream, first, out)
        got = out.cpu().numpy().view(np.uint32)
        np.testing.assert_array_equal(got, ph.words(seed, stream, first, cnt))


@pytest.mark.parametrize("name", ["C1", "C2s", "C3s", "C4s", "C5s"])
def test_generate_matches_host_generator(P, ctx, name):
    import torch
    w = C.SMALL[name]
    s = w.spec
    Xs = G.dataset(s)
    mu = G.column_mean(s)
    elt = 4 if s.dtype == "f32" else 2
    ld = s.d + (-s.d) % (16 // elt)
    X = torch.zeros((s.n, ld), dtype=torch.float32 if s.dtype == "f32" else torch.bfloat16, device="cuda")
    n_local, mu_gpu = P.ppca_generate(ctx, P.gen_spec(s), X)
    assert n_local == s.n
    np.testing.assert_allclose(mu_gpu, mu, rtol=1e-9, atol=1e-12)
    if s.dtype == "f32":
        got = X[:, : s.d].cpu().numpy()
        ulp = np.spacing(np.abs(Xs).astype(np.float32))
        diff = np.abs(got - Xs)
        assert np.all(diff <= ulp), f"max diff in ulps {np.max(diff / ulp)}"
        assert np.mean(diff > 0) < 1e-3
    else:
        got = X[:, : s.d].contiguous().view(torch.int16).cpu().numpy().view(np.uint16)
        gd, hd = G.bf16_bits_to_f64(got), G.bf16_bits_to_f64(Xs)
        assert np.all(np.abs(gd - hd) <= np.spacing(np.abs(hd).astype(np.float32)) * 2 ** 16)
        assert np.mean(got != Xs) < 1e-3


def _split_ref(x32):
    """Host reference of the split layout: hi = RN_bf16(x), lo = RN_bf16(x − hi) (x − hi exact in fp64)."""
    x = x32.astype(np.float64)
    hi = G.f64_to_bf16_bits(x)
    lo = G.f64_to_bf16_bits(x - G.bf16_bits_to_f64(hi))
    return hi, lo


def test_split_f32_bit_exact_and_ragged(P, ctx):
    import torch
    rng = np.random.default_rng(12)
    n, d, ld = 37, 72, 80                               # ragged rows, padded stride
    x = (rng.standard_normal((n, d)) * np.exp(rng.uniform(-20, 20, (n, d)))).astype(np.float32)
    x[0, :4] = [0.0, -0.0, 1e-30, -3.0e38]              # zero, signed zero, tiny, large
    Xd = torch.zeros((n, ld), dtype=torch.float32, device="cuda")
    Xd[:, :d] = torch.from_numpy(x).cuda()
    P.ppca_split_f32(ctx, Xd, d)
    raw = Xd.cpu().numpy().view(np.uint16).reshape(n, 2 * ld)
    hi, lo = _split_ref(x)
    np.testing.assert_array_equal(raw[:, :d], hi)
    np.testing.assert_array_equal(raw[:, d:2 * d], lo)
    # the pair represents x to 2^-17 relative
    rec = G.bf16_bits_to_f64(hi) + G.bf16_bits_to_f64(lo)
    ok = np.abs(x) > 1e-30
    assert np.max(np.abs(rec[ok] - x[ok]) / np.abs(x[ok])) <= 2.0 ** -16
    with pytest.raises(P.PPCAError):
        P.ppca_split_f32(ctx, torch.zeros((4, 20), device="cuda"), 20)   # d % 8 != 0
    P.ppca_split_f32(ctx, torch.zeros((0, 16), device="cuda"), 16)      # empty shard is a no-op


def test_generate_split_equals_split_of_generate(P, ctx):
    import torch
    s = C.SMALL["C3s"].spec
    A = torch.zeros((s.n, s.d), dtype=torch.float32, device="cuda")
    B = torch.zeros_like(A)
    P.ppca_generate(ctx, P.gen_spec(s), A)
    P.ppca_split_f32(ctx, A, s.d)
    P.ppca_generate(ctx, P.gen_spec(s, split=True), B)
    assert torch.equal(A.view(torch.int32), B.view(torch.int32))


# ----------------------------------------------------------------------------- power priming + refine
@pytest.fixture
def impl(P, ctx, request):
    P.ppca_set_pass_impl(ctx, request.param)
    yield request.param
    P.ppca_set_pass_impl(ctx, 0)


def _device_matrix(P, ctx, Xs, spec, split):
    """Stored host X → device ppca_matrix; split=True converts the fp32 rows in place to the
    PPCA_F32_SPLIT layout through the C ABI (ppca_split_f32)."""
    Xd = U.upload(Xs, spec.dtype)
    if split:
        P.ppca_split_f32(ctx, Xd, spec.d)
    return P.matrix(Xd, d=spec.d, split=split)


@pytest.mark.parametrize("split", [False, True], ids=["f32", "split"])
@pytest.mark.parametrize("impl", [1, 2, 3], indirect=True, ids=["simt", "tcgen05", "tcgen05-2kernel"])
@pytest.mark.parametrize("name", ["C1", "C3s", "C5s"])
def test_power_priming_and_refine_parity(P, ctx, name, impl, split):
    """impl 2 runs the single-read fused power pass where eligible (split/bf16 X, m ≤ 64, d ≤ 1024: C3s
    split); impl 3 forces the two-kernel pass."""
    import torch
    if impl >= 2 and name == "C1" and not split:
        pytest.skip("plain-f32 tcgen05 on C1: test_gpu_r2.test_c1_forced_tcgen05_plain_f32_error_budget (R30)")
    w = C.SMALL[name]
    s = w.spec
    if split and s.dtype != "f32":
        pytest.skip("the split layout is for fp32 data")
    Xs, X64 = _host(w)
    lam, T = O.truth(X64)
    W0 = G.init_gaussians(w.init_seed, w.m, s.d)
    W_ref, S_hist = O.prime_power(X64, W0, w.iters)
    E_ref, th_ref, th_all_ref, _ = O.ppca_refine(X64, W_ref, w.k)

    Xm = _device_matrix(P, ctx, Xs, s, split)
    W = torch.zeros((w.m, s.d), dtype=torch.float32, device="cuda")
    th_hist = P.ppca_prime_power(ctx, Xm, w.m, w.iters, w.init_seed, W, theta_hist=True)
    assert P.ppca_last_pass_impl(ctx) == min(impl, 2)
    Wh = W.cpu().numpy().astype(np.float64)
    np.testing.assert_allclose(Wh @ Wh.T, np.eye(w.m), atol=5e-6)
    # the primed subspace equals the oracle's (largest principal angle)
    sv = np.linalg.svd(Wh @ W_ref.T, compute_uv=False)
    assert sv.min() > 1 - 1e-4
    # pPCA-for-free eigenvalues of every iterate (S_t from the same pass) match the oracle's
    worst = 0.0
    for t in range(w.iters):
        ref = O.ritz_values(S_hist[t])
        err_t = U.ritz_rel_err(th_hist[t], ref)
        worst = max(worst, err_t)
        assert err_t < _tol(s), f"iteration {t}"
    print(f"\n[parity] {name} impl={impl} split={split}: per-iteration Ritz rel err max {worst:.3e} (tol {_tol(s)})")
    E = torch.zeros((w.k, s.d), dtype=torch.float32, device="cuda")
    th, dim = P.ppca_refine(ctx, Xm, W, w.m, w.k, E)
    assert dim == w.m
    err = U.assert_ppca_parity(E.cpu().numpy(), th, E_ref, th_ref, T, _tol(s), name, th_all_ref)
    print(f"[parity] {name} impl={impl} split={split}: refine Ritz rel err {err:.3e}")
    # Cauchy interlacing of the GPU Ritz values with the true spectrum
    d, m = s.d, w.m
    for i in range(w.k):
        assert lam[i + d - m] * (1 - _tol(s)) <= th[i] <= lam[i] * (1 + _tol(s))


# ----------------------------------------------------------------------------- minibatch primings
@pytest.mark.parametrize("impl", [0, 1, 2], indirect=True, ids=["auto", "simt", "tcgen05"])
@pytest.mark.parametrize("split", [False, True], ids=["f32", "split"])
def test_oja_parity_c2s(P, ctx, split, impl):
    """C2s (ragged last minibatch: 12096 = 47·256 + 64): auto = the persistent single-kernel Oja
    (oja_persistent.cu), simt = one launch sequence per step, tcgen05 = the tensor-core window pass."""
    import torch
    w = C.SMALL["C2s"]
    s = w.spec
    Xs, X64 = _host(w)
    lam, T = O.truth(X64)
    steps = w.steps
    W_ref, vel_ref = O.prime_oja(X64, G.init_gaussians(w.init_seed, w.m, s.d), w.batch, w.alpha, w.momentum, steps)
    E_ref, th_ref, th_all_ref, _ = O.ppca_refine(X64, W_ref, w.k)
    Xm = _device_matrix(P, ctx, Xs, s, split)
    W = torch.zeros((w.m, s.d), dtype=torch.float32, device="cuda")
    vel = torch.zeros_like(W)
    nxt = P.ppca_prime_oja(ctx, Xm, w.m, w.batch, w.alpha, w.momentum, steps, w.init_seed, W, vel, 0)
    assert nxt == steps
    Wh = W.cpu().numpy().astype(np.float64)
    rel = np.linalg.norm(Wh - W_ref) / np.linalg.norm(W_ref)
    print(f"\n[parity] C2s oja split={split} impl={impl}: trajectory drift {rel:.2e}")
    assert rel < 1e-3, f"Oja trajectory drift {rel:.2e}"
    E = torch.zeros((w.k, s.d), dtype=torch.float32, device="cuda")
    th, dim = P.ppca_refine(ctx, Xm, W, w.m, w.k, E)
    U.assert_ppca_parity(E.cpu().numpy(), th, E_ref, th_ref, T, _tol(s), "C2s", th_all_ref)


@pytest.mark.parametrize("k,batch,d,dtype,split", [
    (10, 100, 200, "f32", False),     # m = 20: components not a multiple of 8, ragged windows (n % b = 7)
    (24, 256, 136, "f32", True),      # m = 48 > 32: two lanes' worth of components per row; split planes
    (16, 64, 784, "bf16", False),     # bf16 storage, many short windows
], ids=["m20-b100-f32", "m48-b256-split", "m32-b64-bf16"])
def test_oja_persistent_shapes(P, ctx, k, batch, d, dtype, split):
    """The persistent single-kernel Oja (auto pass selection, one GPU) on shapes the configs do not
    exercise, against the fp64 oracle's trajectory (same seeded data, init and schedule)."""
    import dataclasses
    import torch
    base = C.SMALL["C2s"]
    spec = dataclasses.replace(base.spec, n=4007, d=d, dtype=dtype)
    w = dataclasses.replace(base, k=k, l=k, batch=batch, spec=spec, steps=90)
    Xs, X64 = _host(w)
    W_ref, _ = O.prime_oja(X64, G.init_gaussians(w.init_seed, w.m, d), w.batch, w.alpha, w.momentum, w.steps)
    Xm = _device_matrix(P, ctx, Xs, spec, split)
    W = torch.zeros((w.m, d), dtype=torch.float32, device="cuda")
    vel = torch.zeros_like(W)
    assert P.ppca_prime_oja(ctx, Xm, w.m, w.batch, w.alpha, w.momentum, w.steps, w.init_seed, W, vel, 0) == w.steps
    rel = np.linalg.norm(W.cpu().numpy().astype(np.float64) - W_ref) / np.linalg.norm(W_ref)
    print(f"\n[parity] oja persistent m={w.m} b={batch} d={d} {dtype}{' split' if split else ''}: drift {rel:.2e}")
    assert rel < 1e-3


def test_oja_persistent_resume_bit_exact(P, ctx):
    """The persistent Oja kernel is deterministic and resumable: 200 steps in one call equal 77 + 123 steps
    through step_io (same W and velocity bits), and the step counter wraps over the epoch boundary."""
    import torch
    w = C.SMALL["C2s"]
    s = w.spec
    Xs, _ = _host(w)
    Xm = _device_matrix(P, ctx, Xs, s, True)
    outs = []
    for chunks in ([200], [77, 123]):
        W = torch.zeros((w.m, s.d), dtype=torch.float32, device="cuda")
        vel = torch.zeros_like(W)
        step = 0
        for i, c in enumerate(chunks):
            step = P.ppca_prime_oja(ctx, Xm, w.m, w.batch, w.alpha, w.momentum, c, w.init_seed if i == 0 else 0,
                                    W, vel, step)
        assert step == 200
        outs.append((W.cpu().numpy(), vel.cpu().numpy()))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("impl", [0, 2], indirect=True, ids=["auto", "tcgen05"])
@pytest.mark.parametrize("split", [False, True], ids=["f32", "split"])
def test_eigengame_parity_c4s(P, ctx, split, impl):
    import torch
    w = C.SMALL["C4s"]
    s = w.spec
    Xs, X64 = _host(w)
    lam, T = O.truth(X64)
    steps = w.steps
    V_ref, _ = O.prime_eigengame(X64, G.init_gaussians(w.init_seed, w.m, s.d), w.batch, w.alpha, w.momentum, steps)
    E_ref, th_ref, th_all_ref, _ = O.ppca_refine(X64, V_ref, w.k)
    Xm = _device_matrix(P, ctx, Xs, s, split)
    V = torch.zeros((w.m, s.d), dtype=torch.float32, device="cuda")
    vel = torch.zeros_like(V)
    P.ppca_prime_eigengame(ctx, Xm, w.m, w.batch, w.alpha, w.momentum, steps, w.init_seed, V, vel, 0)
    if impl == 2 and split:
        assert P.ppca_last_pass_impl(ctx) == 2          # the step's products ran on the tensor cores
    Vh = V.cpu().numpy().astype(np.float64)
    np.testing.assert_allclose(np.linalg.norm(Vh, axis=1), 1, atol=1e-5)
    rel = np.linalg.norm(Vh - V_ref) / np.linalg.norm(V_ref)
    print(f"\n[parity] C4s eigengame split={split} impl={impl}: trajectory drift {rel:.2e}")
    assert rel < 1e-3, f"EigenGame trajectory drift {rel:.2e}"
    E = torch.zeros((w.k, s.d), dtype=torch.float32, device="cuda")
    th, dim = P.ppca_refine(ctx, Xm, V, w.m, w.k, E)
    U.assert_ppca_parity(E.cpu().numpy(), th, E_ref, th_ref, T, _tol(s), "C4s", th_all_ref)


@pytest.mark.parametrize("split", [False, True], ids=["f32", "split"])
@pytest.mark.parametrize("impl", [1, 2], indirect=True, ids=["simt", "tcgen05"])
@pytest.mark.parametrize("name", ["C2s", "C4s"])
def test_refine_parity_random_priming(P, ctx, name, impl, split):
    """Refine (Alg. 1 steps 2–5) of a perturbed-truth priming on the minibatch workloads' data."""
    import torch
    w = C.SMALL[name]
    s = w.spec
    Xs, X64 = _host(w)
    lam, T = O.truth(X64)
    rng = np.random.default_rng(7)
    V = T[: w.m] + 0.05 * rng.standard_normal((w.m, s.d)) / math.sqrt(s.d)
    V32 = V.astype(np.float32)
    E_ref, th_ref, th_all_ref, _ = O.ppca_refine(X64, V32.astype(np.float64), w.k)
    Xm = _device_matrix(P, ctx, Xs, s, split)
    E = torch.zeros((w.k, s.d), dtype=torch.float32, device="cuda")
    th, dim = P.ppca_refine(ctx, Xm, torch.from_numpy(V32).cuda(), w.m, w.k, E)
    assert P.ppca_last_pass_impl(ctx) == impl and dim == w.m
    U.assert_ppca_parity(E.cpu().numpy(), th, E_ref, th_ref, T, _tol(s), name, th_all_ref)


@pytest.mark.parametrize("impl", [1, 2], indirect=True, ids=["simt", "tcgen05"])
@pytest.mark.parametrize("fraction", [0.1, 0.5])
def test_refine_sampled_parity_c3s(P, ctx, impl, fraction):
    """Row-subsampled refine (P L378, R25): the same seeded row tiles on both sides."""
    import torch
    w = C.SMALL["C3s"]
    s = w.spec
    Xs, X64 = _host(w)
    lam, T = O.truth(X64)
    rng = np.random.default_rng(17)
    V32 = (T[: w.m] + 0.05 * rng.standard_normal((w.m, s.d)) / math.sqrt(s.d)).astype(np.float32)
    E_ref, th_ref, used_ref = O.ppca_refine_sampled(X64, V32.astype(np.float64), w.k, fraction, 99)
    Xm = _device_matrix(P, ctx, Xs, s, impl == 2)
    E = torch.zeros((w.k, s.d), dtype=torch.float32, device="cuda")
    th, dim, used = P.ppca_refine_sampled(ctx, Xm, torch.from_numpy(V32).cuda(), w.m, w.k, E, fraction, 99)
    assert used == used_ref and dim == w.m
    assert P.ppca_last_pass_impl(ctx) == impl
    err = U.ritz_rel_err(th, th_ref)
    print(f"\n[parity] C3s sampled refine f={fraction} impl={impl}: rows {used}, Ritz rel err {err:.3e}")
    assert err < 1e-4
    gi = U.gapped(th_ref, w.k)
    assert U.abs_cos(E.cpu().numpy()[gi], E_ref[gi]).min() >= 0.9999
    l_gpu, _ = U.lces_all(E.cpu().numpy(), T[: w.k])          # the paper's measure (P L411-413): identical
    l_ref, _ = U.lces_all(E_ref, T[: w.k])
    assert l_gpu == l_ref, f"sampled refine LCES {l_gpu} vs oracle {l_ref}"


# ----------------------------------------------------------------------------- refine edge cases
def test_refine_counterexample_on_gpu(P, ctx):
    """§4.1 (P L195–228) through the C ABI: d = 3 (row stride padded to 4)."""
    import torch
    X = np.array([[3, 0, 0], [-3, 0, 0], [0, 2, 0], [0, -2, 0], [0, 0, 1], [0, 0, -1]], dtype=np.float32)
    eps = 0.01
    V = np.array([[eps, 0, math.sqrt(1 - eps ** 2)], [0, 1, 0]], dtype=np.float32)
    Xd = U.upload(X, "f32")
    assert Xd.stride(0) == 4
    Xm = P.matrix(Xd, d=3)
    Vd = torch.from_numpy(V).cuda()
    E = torch.zeros((2, 3), dtype=torch.float32, device="cuda")
    th, dim = P.ppca_refine(ctx, Xm, Vd, 2, 2, E)
    Eh = E.cpu().numpy()
    np.testing.assert_allclose(Eh[0], [0, 1, 0], atol=1e-6)
    np.testing.assert_allclose(Eh[1], [eps, 0, math.sqrt(1 - eps ** 2)], atol=1e-6)
    np.testing.assert_allclose(th / 6, [4 / 3, (9 * eps ** 2 + (1 - eps ** 2)) / 3], rtol=1e-6)
    var = P.ppca_captured_variance(ctx, Xm, torch.tensor([[1.0, 0, 0]], device="cuda"), 1)
    assert var[0] == pytest.approx(18.0, rel=1e-7)


def test_refine_full_basis_is_exact_pca_and_errors(P, ctx):
    import torch
    rng = np.random.default_rng(5)
    n, d = 777, 24                               # ragged: not a multiple of any tile
    X = (rng.standard_normal((n, d)) * np.exp(-np.arange(d) / 6)).astype(np.float32)
    X64 = X.astype(np.float64)
    lam, T = O.truth(X64)
    Xd = U.upload(X, "f32")
    Xm = P.matrix(Xd)
    Q = np.ascontiguousarray(np.linalg.qr(rng.standard_normal((d, d)))[0].T, dtype=np.float32)
    E = torch.zeros((d, d), dtype=torch.float32, device="cuda")
    th, dim = P.ppca_refine(ctx, Xm, torch.from_numpy(Q).cuda(), d, d, E)
    assert dim == d
    np.testing.assert_allclose(th, lam, rtol=1e-5)
    cos = U.abs_cos(E.cpu().numpy(), T)
    gi = U.gapped(lam, d)
    assert cos[gi].min() > 0.9999
    # m = 1
    E1 = torch.zeros((1, d), dtype=torch.float32, device="cuda")
    th1, _ = P.ppca_refine(ctx, Xm, torch.from_numpy(T[:1].astype(np.float32)).cuda(), 1, 1, E1)
    assert th1[0] == pytest.approx(lam[0], rel=1e-5)
    # duplicated directions collapse: 2 distinct of 3 requested → SUBSPACE_COLLAPSE for k = 3
    Vdup = torch.from_numpy(np.stack([T[0], T[0], T[1]]).astype(np.float32)).cuda()
    E3 = torch.zeros((3, d), dtype=torch.float32, device="cuda")
    with pytest.raises(P.PPCAError) as ei:
        P.ppca_refine(ctx, Xm, Vdup, 3, 3, E3)
    assert ei.value.name == "PPCA_ERR_SUBSPACE_COLLAPSE"
    th2, dim2 = P.ppca_refine(ctx, Xm, Vdup, 3, 2, E3[:2])
    assert dim2 == 2
    # m > d
    with pytest.raises(P.PPCAError) as ei:
        P.ppca_refine(ctx, Xm, torch.zeros((d + 1, d), device="cuda"), d + 1, 1, E)
    assert ei.value.name == "PPCA_ERR_TOO_MANY_COMPONENTS"


def test_eval_and_captured_variance(P, ctx):
    import torch
    rng = np.random.default_rng(6)
    k, d = 5, 40
    T = np.ascontiguousarray(np.linalg.qr(rng.standard_normal((d, k)))[0].T)
    E = T + 1e-3 * rng.standard_normal((k, d)) * np.array([[0.1], [1], [5], [0.1], [0.1]])
    E /= np.linalg.norm(E, axis=1, keepdims=True)
    Et = torch.from_numpy(E.astype(np.float32)).cuda()
    Tt = torch.from_numpy(T.astype(np.float32)).cuda()
    ang, lc = P.ppca_eval(ctx, Et, Tt, k, d, U.THRESHOLDS)
    ref = O.angles(E.astype(np.float32).astype(np.float64), T.astype(np.float32).astype(np.float64))
    np.testing.assert_allclose(ang, ref, atol=1e-6)
    assert lc.tolist() == [O.lces(ref, V) for V in U.THRESHOLDS]
    X = rng.standard_normal((301, d)).astype(np.float32)
    Xm = P.matrix(U.upload(X, "f32"))
    var = P.ppca_captured_variance(ctx, Xm, Et, k)
    np.testing.assert_allclose(var, [O.captured_variance(X.astype(np.float64), e) for e in
                                     E.astype(np.float32).astype(np.float64)], rtol=1e-5)
    Gd = torch.zeros((d, d), dtype=torch.float64, device="cuda")
    P.ppca_gram(ctx, Xm, Gd)
    np.testing.assert_allclose(Gd.cpu().numpy(), X.astype(np.float64).T @ X.astype(np.float64), rtol=1e-5, atol=1e-3)


def test_launch_count_and_no_fallback(P, ctx):
    before = P.ppca_launch_count(ctx)
    import torch
    W = torch.zeros((4, 64), device="cuda")
    X = U.upload(np.random.default_rng(0).standard_normal((100, 64)).astype(np.float32), "f32")
    P.ppca_prime_power(ctx, P.matrix(X), 4, 2, 7, W)
    assert P.ppca_launch_count(ctx) > before
