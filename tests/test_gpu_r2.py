"""GPU parity at the shapes the kernels take at full size, the collective call sites, the stop rule and
the certification support (round 2).  Every comparison is against the fp64 oracle on the same seeded
inputs (host generator), with BASELINE.json north_star's tolerances: Ritz values 1e-4 relative (1e-3
for the bf16-stored config), |cos| ≥ 0.9999 where the relative eigengap > 1e-2, identical LCES.

  * C3m: n = 131075 (ragged), d = 1024 = C3's d, m = 64 — the fused single-read power pass with four
    256-column d-groups per row group (the cross-CTA flag protocol full-size C3 runs);
  * C4m: d = 4096 = C4's d — the two-kernel power pass (kernel A2 + kernel B, d > 1024) and the
    EigenGame window pass;
  * C5m: d = 65536 = C5's d, bf16, m = 128 — kernel A2 on 2-CTA pairs and the lean kernel B;
  * a one-rank NCCL communicator: every all-reduce call site of the path runs and leaves results bitwise
    identical; the paper's stop rule (P L61-62); residual certification (reading R29).
"""
import dataclasses
import math
import os

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


def _device(P, ctx, Xs, spec, split):
    Xd = U.upload(Xs, spec.dtype)
    if split:
        P.ppca_split_f32(ctx, Xd, spec.d)
    return P.matrix(Xd, d=spec.d, split=split)


def _top_truth(X64, k):
    """Top-k eigenpairs of XᵀX (library eigensolver on the formed fp64 Gram; test infrastructure)."""
    import scipy.linalg
    Cm = X64.T @ X64
    d = Cm.shape[0]
    w, V = scipy.linalg.eigh(Cm, subset_by_index=[d - k - 1, d - 1])
    order = np.argsort(-w, kind="stable")
    return w[order], O.sign_convention(V[:, order].T)


def _power_parity(P, ctx, Xm, X64, w, iters, T=None, check_kernels=None):
    """Power priming + refine on the device vs the oracle: per-iterate Ritz values, the primed subspace, refine
    Ritz values / vectors, LCES (when the truth T is given)."""
    import torch
    s = w.spec
    W0 = G.init_gaussians(w.init_seed, w.m, s.d)
    W_ref, S_hist = O.prime_power(X64, W0, iters)
    E_ref, th_ref, th_all_ref, _ = O.ppca_refine(X64, W_ref, w.k)
    W = torch.zeros((w.m, s.d), dtype=torch.float32, device="cuda")
    P.ppca_set_timing(ctx, True)
    P.ppca_get_kernel_time(ctx, 0), P.ppca_get_kernel_time(ctx, 1)
    th_hist = P.ppca_prime_power(ctx, Xm, w.m, iters, w.init_seed, W, theta_hist=True)
    ka = P.ppca_get_kernel_time(ctx, 0)[1]
    kb = P.ppca_get_kernel_time(ctx, 1)[1]
    P.ppca_set_timing(ctx, False)
    if check_kernels is not None:
        check_kernels(ka, kb)
    worst = 0.0
    for t in range(iters):
        e = U.ritz_rel_err(th_hist[t], O.ritz_values(S_hist[t]))
        worst = max(worst, e)
        assert e < _tol(s), f"{w.name} iteration {t}: {e:.3e}"
    Wh = W.cpu().numpy().astype(np.float64)
    assert np.linalg.svd(Wh @ W_ref.T, compute_uv=False).min() > 1 - 1e-4
    E = torch.zeros((w.k, s.d), dtype=torch.float32, device="cuda")
    th, dim = P.ppca_refine(ctx, Xm, W, w.m, w.k, E)
    assert dim == w.m
    Eh = E.cpu().numpy()
    err = U.ritz_rel_err(th, th_ref)
    assert err < _tol(s), f"{w.name} refine: {err:.3e}"
    gi = U.gapped(th_all_ref, w.k)
    if gi.size:
        assert U.abs_cos(Eh[gi], E_ref[gi]).min() >= 0.9999
    if T is not None:
        l_gpu, _ = U.lces_all(Eh, T[: w.k])
        l_ref, _ = U.lces_all(E_ref, T[: w.k])
        assert l_gpu == l_ref, f"{w.name}: LCES {l_gpu} vs oracle {l_ref}"
    print(f"\n[parity] {w.name}: per-iterate Ritz err {worst:.2e}, refine {err:.2e} (tol {_tol(s)})")
    return W


# ----------------------------------------------------------------------------- full-width shapes
C3M = dataclasses.replace(C.C3, name="C3m", spec=dataclasses.replace(C.C3.spec, n=131_075), iters=6)
C4M = dataclasses.replace(C.C4, name="C4m", spec=dataclasses.replace(C.C4.spec, n=12_300), steps=6)
C5M = dataclasses.replace(C.C5, name="C5m", spec=dataclasses.replace(C.C5.spec, n=6_007), iters=3)


@pytest.mark.parametrize("impl", [0, 4], ids=["pair", "rowgroup"])
def test_c3m_fused_pass_vs_oracle(P, ctx, impl):
    """d = 1024, the launch configuration of full-size C3, against the oracle: impl 0 (auto) runs the d-sliced
    pair kernel (two 512-column slices per row group, Y exchanged through distributed shared memory); impl 4
    the row-group kernel (4 d-groups per row group, per-tile flags, Y rows through global memory, X_hi re-read
    from L2 by the siblings)."""
    w = C3M
    Xs = G.dataset(w.spec)
    X64 = G.stored_to_f64(Xs, w.spec.dtype)
    lam, T = _top_truth(X64, w.k)
    Xm = _device(P, ctx, Xs, w.spec, True)
    P.ppca_set_pass_impl(ctx, impl)

    def only_fused(ka, kb):
        assert ka == w.iters and kb == 0, f"expected the single-read fused kernel only (A {ka}, B {kb})"

    try:
        _power_parity(P, ctx, Xm, X64, w, w.iters, T, only_fused)
        assert P.ppca_last_power_kernel(ctx) == (4 if impl == 0 else 3)
    finally:
        P.ppca_set_pass_impl(ctx, 0)


PAIR_RAGGED = [
    # split fp32, d = 800: slice 1 holds 288 columns (5 chunks, 3 d-chunks of 128, the last one partial)
    dataclasses.replace(C.C3, name="C3r", spec=dataclasses.replace(C.C3.spec, n=40_007, d=800), iters=4),
    # bf16, d = 576: slice 1 holds 64 columns (1 chunk, 1 d-chunk); a ragged last row tile
    dataclasses.replace(C.C5, name="C5r", k=32, l=32, spec=dataclasses.replace(C.C5.spec, n=9_001, d=576), iters=3),
]


@pytest.mark.parametrize("w", PAIR_RAGGED, ids=[x.name for x in PAIR_RAGGED])
def test_pair_pass_ragged_slices_vs_oracle(P, ctx, w):
    """The d-sliced pair kernel where the second slice is partial (d not a multiple of 512) and the row count
    is not a multiple of the 128-row tile, against the oracle."""
    Xs = G.dataset(w.spec)
    X64 = G.stored_to_f64(Xs, w.spec.dtype)
    lam, T = _top_truth(X64, w.k)
    Xm = _device(P, ctx, Xs, w.spec, w.spec.dtype == "f32")
    P.ppca_set_pass_impl(ctx, 2)                 # the tensor-core path even where auto picks the CUDA cores
    try:
        _power_parity(P, ctx, Xm, X64, w, w.iters, T,
                      lambda ka, kb: (ka == w.iters and kb == 0) or pytest.fail(f"A {ka} B {kb}"))
    finally:
        P.ppca_set_pass_impl(ctx, 0)


def test_c3m_two_kernel_pass_matches_oracle(P, ctx):
    """The same shape through the two-kernel pass (kernel A2 + kernel B) — the fallback of the fused kernel."""
    impl = 3
    w = C3M
    Xs = G.dataset(w.spec)
    X64 = G.stored_to_f64(Xs, w.spec.dtype)
    Xm = _device(P, ctx, Xs, w.spec, True)
    P.ppca_set_pass_impl(ctx, impl)
    try:
        _power_parity(P, ctx, Xm, X64, w, 4, None, lambda ka, kb: (ka == 4 and kb == 4) or pytest.fail(f"{ka} {kb}"))
    finally:
        P.ppca_set_pass_impl(ctx, 0)


@pytest.fixture(scope="module")
def c4m(P, ctx):
    w = C4M
    Xs = G.dataset(w.spec)
    X64 = G.stored_to_f64(Xs, w.spec.dtype)
    lam, T = _top_truth(X64, w.k)
    return w, Xs, X64, T


def test_c4m_d4096_two_kernel_power_vs_oracle(P, ctx, c4m):
    """d = 4096 (C4's d, beyond the fused kernel's one-segment rule): kernel A2 + kernel B power passes."""
    w, Xs, X64, T = c4m
    Xm = _device(P, ctx, Xs, w.spec, True)
    P.ppca_set_pass_impl(ctx, 0)
    pw = dataclasses.replace(w, priming="power")
    _power_parity(P, ctx, Xm, X64, pw, 4, T, lambda ka, kb: (ka == 4 and kb == 4) or pytest.fail(f"{ka} {kb}"))


def test_c4m_d4096_eigengame_window_vs_oracle(P, ctx, c4m):
    """d = 4096, batch 4096: the EigenGame step's tensor-core window pass (K-split over the SMs) + the
    cooperative update, the trajectory and the refine against the oracle."""
    import torch
    w, Xs, X64, T = c4m
    Xm = _device(P, ctx, Xs, w.spec, True)
    V_ref, _ = O.prime_eigengame(X64, G.init_gaussians(w.init_seed, w.m, w.spec.d), w.batch, w.alpha, w.momentum,
                                 w.steps)
    E_ref, th_ref, th_all_ref, _ = O.ppca_refine(X64, V_ref, w.k)
    V = torch.zeros((w.m, w.spec.d), dtype=torch.float32, device="cuda")
    vel = torch.zeros_like(V)
    P.ppca_prime_eigengame(ctx, Xm, w.m, w.batch, w.alpha, w.momentum, w.steps, w.init_seed, V, vel, 0)
    assert P.ppca_last_pass_impl(ctx) == 2
    rel = np.linalg.norm(V.cpu().numpy().astype(np.float64) - V_ref) / np.linalg.norm(V_ref)
    assert rel < 1e-3, f"EigenGame drift {rel:.2e}"
    E = torch.zeros((w.k, w.spec.d), dtype=torch.float32, device="cuda")
    th, _ = P.ppca_refine(ctx, Xm, V, w.m, w.k, E)
    U.assert_ppca_parity(E.cpu().numpy(), th, E_ref, th_ref, T, _tol(w.spec), "C4m", th_all_ref)
    print(f"\n[parity] C4m eigengame: drift {rel:.2e}")


def test_c5m_full_width_bf16_vs_oracle(P, ctx):
    """d = 65536 (C5's d), bf16, m = 128: kernel A2 on 2-CTA pairs and the lean kernel B of the full-size
    config, per-iterate Ritz values and the refine against the oracle (1e-3, bf16-stored config)."""
    w = C5M
    Xs = G.dataset(w.spec)
    X64 = G.stored_to_f64(Xs, w.spec.dtype)
    Xm = _device(P, ctx, Xs, w.spec, False)
    del Xs
    P.ppca_set_pass_impl(ctx, 0)
    _power_parity(P, ctx, Xm, X64, w, w.iters, None,
                  lambda ka, kb: (ka == w.iters and kb == w.iters) or pytest.fail(f"{ka} {kb}"))


# ----------------------------------------------------------------------------- forced tcgen05 on C1 (R30)
def test_c1_forced_tcgen05_split_is_within_bar(P, ctx):
    """C1 (n = 2000) on the tensor cores with the split layout: below 32768 rows product 2 adds X_lo·Y_hi
    (reading R30), so the per-iterate and refine Ritz values meet the 1e-4 bar and LCES agree."""
    w = C.C1
    Xs = G.dataset(w.spec)
    X64 = G.stored_to_f64(Xs, w.spec.dtype)
    lam, T = O.truth(X64)
    Xm = _device(P, ctx, Xs, w.spec, True)
    P.ppca_set_pass_impl(ctx, 2)
    try:
        _power_parity(P, ctx, Xm, X64, w, w.iters, T)
        assert P.ppca_last_pass_impl(ctx) == 2
    finally:
        P.ppca_set_pass_impl(ctx, 0)


def test_c1_forced_tcgen05_plain_f32_error_budget(P, ctx):
    """PPCA_F32 (not split) on the tensor cores rounds X to bf16 in product 2 (reading R30): the documented
    budget is 1e-3 relative on C1's Ritz values (auto keeps such shards on the exact-fp32 CUDA-core pass)."""
    import torch
    w = C.C1
    Xs = G.dataset(w.spec)
    X64 = G.stored_to_f64(Xs, w.spec.dtype)
    W_ref, S_hist = O.prime_power(X64, G.init_gaussians(w.init_seed, w.m, w.spec.d), w.iters)
    Xm = _device(P, ctx, Xs, w.spec, False)
    P.ppca_set_pass_impl(ctx, 2)
    try:
        W = torch.zeros((w.m, w.spec.d), dtype=torch.float32, device="cuda")
        th = P.ppca_prime_power(ctx, Xm, w.m, w.iters, w.init_seed, W, theta_hist=True)
    finally:
        P.ppca_set_pass_impl(ctx, 0)
    worst = max(U.ritz_rel_err(th[t], O.ritz_values(S_hist[t])) for t in range(w.iters))
    print(f"\n[R30] C1 plain-f32 tcgen05: per-iterate Ritz err {worst:.2e}")
    assert worst < 1e-3


# ----------------------------------------------------------------------------- collectives on one GPU
def test_one_rank_nccl_comm_runs_every_allreduce_bitwise(P):
    """A world-1 context with a one-rank NCCL communicator runs every collective call site of the path (grouped
    [Z|S] per power iteration and per minibatch step, S of the refine, the row count of the sampled refine,
    the generator's column mean); the results are bitwise those of a context without one."""
    import torch
    stream = torch.cuda.current_stream()
    plain = P.ppca_ctx_create(0, stream)
    comm = P.ppca_ctx_create_one_rank_comm(0, stream)
    try:
        w = C.SMALL["C3s"]
        s = w.spec
        outs = []
        for h in (plain, comm):
            X = torch.empty((s.n, s.d), dtype=torch.float32, device="cuda")
            _, mu = P.ppca_generate(h, P.gen_spec(s, split=True), X)
            Xm = P.matrix(X, split=True)
            c0 = P.ppca_collective_count(h)
            W = torch.zeros((w.m, s.d), dtype=torch.float32, device="cuda")
            th = P.ppca_prime_power(h, Xm, w.m, 5, w.init_seed, W, theta_hist=True)
            c1 = P.ppca_collective_count(h)
            E = torch.zeros((w.k, s.d), dtype=torch.float32, device="cuda")
            the, _ = P.ppca_refine(h, Xm, W, w.m, w.k, E)
            ths, _, used = P.ppca_refine_sampled(h, Xm, W, w.m, w.k, E, 0.3, 5)
            outs.append((mu, th, W.cpu().numpy(), the, ths, used, c1 - c0))
        (mu0, th0, W0, e0, s0, u0, n0), (mu1, th1, W1, e1, s1, u1, n1) = outs
        assert n0 == 0 and n1 == 5, f"collectives: plain {n0}, comm {n1}"
        assert np.array_equal(mu0, mu1) and np.array_equal(th0, th1) and np.array_equal(W0, W1)
        assert np.array_equal(e0, e1) and np.array_equal(s0, s1) and u0 == u1
        # minibatch steps: one grouped all-reduce per step (the per-step launch sequence)
        w2 = C.SMALL["C2s"]
        s2 = w2.spec
        res = []
        for h in (plain, comm):
            P.ppca_set_pass_impl(h, 1)                     # same kernels on both (the persistent Oja is 1-GPU only)
            X = torch.empty((s2.n, s2.d), dtype=torch.float32, device="cuda")
            P.ppca_generate(h, P.gen_spec(s2), X)
            Xm = P.matrix(X)
            V = torch.zeros((w2.m, s2.d), dtype=torch.float32, device="cuda")
            vel = torch.zeros_like(V)
            c0 = P.ppca_collective_count(h)
            P.ppca_prime_oja(h, Xm, w2.m, w2.batch, w2.alpha, w2.momentum, 20, w2.init_seed, V, vel, 0)
            P.ppca_prime_eigengame(h, Xm, w2.m, w2.batch, 1e-4, 0.9, 7, w2.init_seed, V, vel, 0)
            res.append((V.cpu().numpy(), vel.cpu().numpy(), P.ppca_collective_count(h) - c0))
        assert res[0][2] == 0 and res[1][2] >= 27
        assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[0][1], res[1][1])
    finally:
        P.ppca_ctx_destroy(plain)
        P.ppca_ctx_destroy(comm)


def _two_gpu_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    import paper_2109_03709_b200 as P
    P.load()
    h = P.ppca_ctx_create_distributed(rank, torch.cuda.current_stream())
    w = C.SMALL["C3s"]
    s = w.spec
    _, n_local = P.contiguous_shard(s.n, rank, world)
    X = torch.empty((n_local, s.d), dtype=torch.float32, device="cuda")
    P.ppca_generate(h, P.gen_spec(s, split=True), X)
    Xm = P.matrix(X, n_global=s.n, split=True)
    W = torch.zeros((w.m, s.d), dtype=torch.float32, device="cuda")
    th = P.ppca_prime_power(h, Xm, w.m, w.iters, w.init_seed, W, theta_hist=True)
    q.put((rank, th, W.cpu().numpy()))
    P.ppca_ctx_destroy(h)
    dist.destroy_process_group()


def test_two_gpus_power_priming_bitwise_identical_across_ranks_and_matches_oracle():
    """Two ranks over NCCL (skipped with fewer than 2 GPUs): θ history and W bitwise identical on both ranks,
    per-iterate Ritz values within 1e-4 of the oracle (contiguous row shards, reading R10 / §6)."""
    import torch
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    ctxmp = mp.get_context("spawn")
    q = ctxmp.Queue()
    port = 29000 + os.getpid() % 1000
    procs = [ctxmp.Process(target=_two_gpu_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict((r, (th, W)) for r, th, W in (q.get(timeout=600) for _ in procs))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert np.array_equal(got[0][0], got[1][0]) and np.array_equal(got[0][1], got[1][1])
    w = C.SMALL["C3s"]
    X64 = G.dataset_f64(w.spec)
    _, S_hist = O.prime_power(X64, G.init_gaussians(w.init_seed, w.m, w.spec.d), w.iters)
    for t in range(w.iters):
        assert U.ritz_rel_err(got[0][0][t], O.ritz_values(S_hist[t])) < 1e-4


# ----------------------------------------------------------------------------- stop rule (P L61-62)
def test_power_stop_rule_matches_oracle(P, ctx):
    """ε chosen between two consecutive column moves of the oracle's trajectory (clear margin): the device
    stops after the same iteration and its θ history matches."""
    import torch
    w = C.SMALL["C3s"]
    s = w.spec
    Xs = G.dataset(s)
    X64 = G.stored_to_f64(Xs, s.dtype)
    W0 = G.init_gaussians(w.init_seed, w.m, s.d)
    W = O.gram_schmidt(O.init_vectors(W0), drop=False)
    moves = []
    for _ in range(10):
        Wn, _ = O.power_step(X64, W)
        moves.append(float(np.max(O.column_moves(Wn, W))))
        W = Wn
    t_stop = next(t for t in range(3, 10) if moves[t] < moves[t - 1] / 1.3)
    eps = math.sqrt(moves[t_stop] * moves[t_stop - 1])
    W_ref, S_hist = O.prime_power(X64, W0, 10, eps=eps)
    assert len(S_hist) == t_stop + 1
    Xm = _device(P, ctx, Xs, s, True)
    Wd = torch.zeros((w.m, s.d), dtype=torch.float32, device="cuda")
    th, done = P.ppca_prime_power_ex(ctx, Xm, w.m, 10, w.init_seed, Wd, theta_hist=True, eps=eps)
    assert done == len(S_hist), f"device stopped after {done}, oracle after {len(S_hist)}"
    for t in range(done):
        assert U.ritz_rel_err(th[t], O.ritz_values(S_hist[t])) < 1e-4
    # eps <= 0: the whole budget
    _, done0 = P.ppca_prime_power_ex(ctx, Xm, w.m, 4, w.init_seed, Wd, eps=0.0)
    assert done0 == 4


# ----------------------------------------------------------------------------- certification (R29)
def test_ritz_residuals_match_oracle_c5s(P, ctx):
    """‖XᵀX e_i − θ_i e_i‖ of the refine's Ritz pairs after 2 power iterations (residuals far above rounding),
    device (exact-fp32 CUDA-core pass) vs the oracle's residuals of its own pairs; and at exact eigenvectors
    of a planted diagonal-like problem the residual is at rounding level."""
    import torch
    w = C.SMALL["C5s"]
    s = w.spec
    Xs = G.dataset(s)
    X64 = G.stored_to_f64(Xs, s.dtype)
    W_ref, _ = O.prime_power(X64, G.init_gaussians(w.init_seed, w.m, s.d), 2)
    k = 16
    E_ref, th_ref, _, _ = O.ppca_refine(X64, W_ref, k)
    r_ref = O.ritz_residuals(X64, E_ref, th_ref)
    Xm = _device(P, ctx, Xs, s, False)
    W = torch.zeros((w.m, s.d), dtype=torch.float32, device="cuda")
    P.ppca_prime_power(ctx, Xm, w.m, 2, w.init_seed, W)
    E = torch.zeros((k, s.d), dtype=torch.float32, device="cuda")
    th, _ = P.ppca_refine(ctx, Xm, W, w.m, k, E)
    r, rg = P.ppca_ritz_residuals(ctx, Xm, E, k, th, gram=True)
    np.testing.assert_allclose(np.sqrt(np.diag(rg)), r, rtol=1e-4)           # the Gram of the same residual rows
    R_ref = (X64 @ E_ref.T).T @ X64 - th_ref[:, None] * E_ref
    assert np.sqrt(np.linalg.eigvalsh(rg)[-1]) == pytest.approx(np.linalg.norm(R_ref, 2), rel=2e-2)
    print(f"\n[R29] C5s residuals / θ1: oracle {np.min(r_ref) / th_ref[0]:.2e} … {np.max(r_ref) / th_ref[0]:.2e}, "
          f"max rel diff {np.max(np.abs(r - r_ref) / r_ref):.2e}")
    np.testing.assert_allclose(r, r_ref, rtol=2e-2)
    assert np.max(r_ref) > 1e-3 * th_ref[0]              # a non-converged block: residuals far above rounding


def test_refine_orthonormal_flag_vs_oracle(P, ctx):
    """ppca_refine_ex(PPCA_REFINE_ORTHONORMAL) on ppca_prime_power's W (orthonormal rows): B = orth(V) skipped,
    the generalized Rayleigh–Ritz keeps θ and E those of span W — against the oracle's refine of its own priming,
    and against the flag-less refine."""
    import torch
    w = C.SMALL["C3s"]
    s = w.spec
    Xs = G.dataset(s)
    X64 = G.stored_to_f64(Xs, s.dtype)
    lam, T = O.truth(X64)
    W_ref, _ = O.prime_power(X64, G.init_gaussians(w.init_seed, w.m, s.d), w.iters)
    E_ref, th_ref, th_all_ref, _ = O.ppca_refine(X64, W_ref, w.k)
    Xm = _device(P, ctx, Xs, s, True)
    W = torch.zeros((w.m, s.d), dtype=torch.float32, device="cuda")
    P.ppca_prime_power(ctx, Xm, w.m, w.iters, w.init_seed, W)
    E = torch.zeros((w.k, s.d), dtype=torch.float32, device="cuda")
    th, dim = P.ppca_refine_ex(ctx, Xm, W, w.m, w.k, E, P.PPCA_REFINE_ORTHONORMAL)
    assert dim == w.m
    U.assert_ppca_parity(E.cpu().numpy(), th, E_ref, th_ref, T, 1e-4, "C3s refine_ex", th_all_ref)
    E2 = torch.zeros_like(E)
    th2, _ = P.ppca_refine(ctx, Xm, W, w.m, w.k, E2)
    assert U.ritz_rel_err(th, th2) < 1e-6
    with pytest.raises(P.PPCAError):
        P.ppca_refine_ex(ctx, Xm, W, w.m, w.k, E, 4)       # unknown flag


def test_theorem1_assertion_vs_oracle(P, ctx):
    """Theorem 1 online assertion (P L308-312, NEXT-4) on the device against the oracle: near-converged primings
    of C3s (V = truth + δ·noise): the same leading run of Prop. 3 conditions, the same angles, and the conclusion
    (pPCA no farther from e_i than the priming on that run) holds on both sides."""
    import torch
    w = C.SMALL["C3s"]
    s = w.spec
    Xs = G.dataset(s)
    X64 = G.stored_to_f64(Xs, s.dtype)
    lam, T = O.truth(X64)
    Xm = _device(P, ctx, Xs, s, True)
    k, m = 8, 16
    Tt = torch.from_numpy(T[:k].astype(np.float32)).cuda()
    for delta in [1e-3, 3e-2]:
        V32 = (T[:m] + delta * np.random.default_rng(3).standard_normal((m, s.d)) / math.sqrt(s.d)).astype(np.float32)
        up_ref, ap_ref, aq_ref, holds_ref = O.theorem1_check(X64, V32.astype(np.float64), T, k, tol=1e-4)
        up, ap, aq, holds = P.ppca_check_theorem1(ctx, Xm, torch.from_numpy(V32).cuda(), m, k, Tt, 1e-4)
        print(f"\n[theorem1] delta {delta}: run {up} (oracle {up_ref}), holds {holds}")
        assert up == up_ref and holds and holds_ref
        # angles from fp32 unit rows (acos of |⟨e, t⟩|): resolved to ~5e-4 near zero
        np.testing.assert_allclose(ap, ap_ref, atol=1e-3)
        np.testing.assert_allclose(aq, aq_ref, atol=1e-3)


# ----------------------------------------------------------------------------- huge d (NEXT-3)
C6M = C.Workload("C6m", G.GenSpec("planted_householder", n=1_100, d=524_288, seed=1005, spectrum="power", a=1.0,
                                  relu=True, house_r=8, dtype="bf16"),
                 k=8, l=0, priming="eigengame", batch=1024, alpha=1e-2, steps=4, init_seed=2005)


def test_huge_d_eigengame_and_refine_vs_oracle(P, ctx):
    """The paper's large-scale regime (P L373-381: d ~ 13M, EigenGame batch 1024, k = 8, pPCA without extra
    components, 10 % projection) at d = 524288 with few rows: K-split window passes (8192 K chunks), 4096
    d-groups in kernel B, the K-split refine pass (fewer row tiles than SMs) and the sampled refine — the same
    kernel paths the 13.1M-dim tool run takes — against the oracle."""
    import torch
    w = C6M
    s = w.spec
    Xs = G.dataset(s)
    X64 = G.stored_to_f64(Xs, s.dtype)
    Xm = _device(P, ctx, Xs, s, False)
    del Xs
    V_ref, _ = O.prime_eigengame(X64, G.init_gaussians(w.init_seed, w.m, s.d), w.batch, w.alpha, w.momentum, w.steps)
    V = torch.zeros((w.m, s.d), dtype=torch.float32, device="cuda")
    vel = torch.zeros_like(V)
    P.ppca_prime_eigengame(ctx, Xm, w.m, w.batch, w.alpha, w.momentum, w.steps, w.init_seed, V, vel, 0)
    Vh = V.cpu().numpy().astype(np.float64)
    rel = np.linalg.norm(Vh - V_ref) / np.linalg.norm(V_ref)
    V0 = O.init_vectors(G.init_gaussians(w.init_seed, w.m, s.d))
    moved = np.linalg.norm(V_ref - V0) / np.linalg.norm(V0)
    print(f"\n[huge-d] d={s.d}: EigenGame drift {rel:.2e} (trajectory moved {moved:.2e})")
    assert rel < 1e-3 and moved > 1e-2
    E_ref, th_ref, th_all_ref, _ = O.ppca_refine(X64, V_ref, w.k)
    E = torch.zeros((w.k, s.d), dtype=torch.float32, device="cuda")
    th, dim = P.ppca_refine(ctx, Xm, V, w.m, w.k, E)
    err = U.ritz_rel_err(th, th_ref)
    print(f"[huge-d] refine Ritz rel err {err:.2e}")
    assert err < 1e-3
    gi = U.gapped(th_all_ref, w.k)
    if gi.size:
        assert U.abs_cos(E.cpu().numpy()[gi], E_ref[gi]).min() >= 0.9999
    # the paper's 10 % projection (P L378, R25): same seeded tiles on both sides
    E2, th2r, used_ref = O.ppca_refine_sampled(X64, V_ref, w.k, 0.5, 77)
    th2, _, used = P.ppca_refine_sampled(ctx, Xm, V, w.m, w.k, E, 0.5, 77)
    assert used == used_ref
    assert U.ritz_rel_err(th2, th2r) < 1e-3


# ----------------------------------------------------------------------------- distributed CholQR (§6)
def _power_run(P, h, s, w, iters, split):
    import torch
    X = torch.empty((s.n, s.d), dtype=torch.bfloat16 if s.dtype == "bf16" else torch.float32, device="cuda")
    P.ppca_generate(h, P.gen_spec(s, split=s.dtype == "f32"), X)
    Xm = P.matrix(X, split=s.dtype == "f32")
    P.ppca_set_orth_split(h, split)
    P.ppca_set_pass_impl(h, 2)
    try:
        W = torch.zeros((w.m, s.d), dtype=torch.float32, device="cuda")
        c0 = P.ppca_collective_count(h)
        th = P.ppca_prime_power(h, Xm, w.m, iters, w.init_seed, W, theta_hist=True)
        return th, W.cpu().numpy(), P.ppca_collective_count(h) - c0
    finally:
        P.ppca_set_orth_split(h, 0)
        P.ppca_set_pass_impl(h, 0)


def test_distributed_orth_nccl_path_one_rank_bitwise(P):
    """The d-sliced CholQR's NCCL path (reduce-scatter of Z + all-reduce of S in one group, slice Gram, m×m
    all-reduce, slice apply, all-gather of W) over a one-rank communicator: bitwise the replicated CholQR, three
    NCCL operations per iteration."""
    import torch
    w = C.SMALL["C5s"]
    s = w.spec
    stream = torch.cuda.current_stream()
    plain = P.ppca_ctx_create(0, stream)
    comm = P.ppca_ctx_create_one_rank_comm(0, stream)
    try:
        th0, W0, n0 = _power_run(P, plain, s, w, 4, 0)
        th1, W1, n1 = _power_run(P, comm, s, w, 4, -1)
    finally:
        P.ppca_ctx_destroy(plain)
        P.ppca_ctx_destroy(comm)
    assert n0 == 0 and n1 == 3 * 4, f"collectives {n0} / {n1}"
    assert np.array_equal(th0, th1) and np.array_equal(W0, W1)


@pytest.mark.parametrize("blocks", [2, 4])
def test_distributed_orth_emulated_slices_match(P, ctx, blocks):
    """b emulated d-slices on one GPU (the blocked Z layout, slice Grams summed, slice applies, the unblocking):
    the same CholQR up to the Gram's summation order, and the oracle's per-iterate Ritz values (C5s, bf16)."""
    w = C.SMALL["C5s"]
    s = w.spec
    th0, W0, _ = _power_run(P, ctx, s, w, 4, 1)
    th1, W1, _ = _power_run(P, ctx, s, w, 4, blocks)
    assert U.ritz_rel_err(th1, th0) < 1e-6
    assert np.max(np.abs(W1 - W0)) < 1e-5
    X64 = G.dataset_f64(s)
    _, S_hist = O.prime_power(X64, G.init_gaussians(w.init_seed, w.m, s.d), 4)
    for t in range(4):
        assert U.ritz_rel_err(th1[t], O.ritz_values(S_hist[t])) < 1e-3


def test_upload_rows_matches_device_split(P, ctx):
    """ppca_upload_rows (the e2e path: host rows → the device shard, split in place) equals the device-side
    ppca_split_f32 of the same rows bit for bit, for a row block at an offset, and for bf16 rows."""
    import torch
    rng = np.random.default_rng(7)
    n, d = 3001, 256
    host = torch.from_numpy(rng.standard_normal((n, d)).astype(np.float32)).pin_memory()
    ref = host.cuda()
    P.ppca_split_f32(ctx, ref, d)
    dev = torch.zeros((n, d), dtype=torch.float32, device="cuda")
    Xm = P.matrix(dev, split=True)
    P.ppca_upload_rows(ctx, host[:1000], Xm, 0)
    P.ppca_upload_rows(ctx, host[1000:], Xm, 1000)
    assert torch.equal(dev.view(torch.int32), ref.view(torch.int32))
    hb = host.to(torch.bfloat16)
    devb = torch.zeros((n, d), dtype=torch.bfloat16, device="cuda")
    P.ppca_upload_rows(ctx, hb, P.matrix(devb), 0)
    assert torch.equal(devb.cpu().view(torch.int16), hb.view(torch.int16))
    with pytest.raises(P.PPCAError):
        P.ppca_upload_rows(ctx, host[:10], Xm, n - 5)          # outside the shard
