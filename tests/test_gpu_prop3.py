"""Prop. 3 checker (P L293–302; S L337–345; reading R28): ppca_check_prop3 through the
C ABI against the fp64 oracle check_prop3 on the same fp32 inputs.

Tolerance: the device orthonormalises V into fp32 rows and forms the projected Gram from fp32 data, so
span S and C' carry ~1e-7 relative perturbations; an angle moves by that over the relative eigengap of
the projected covariance (≥ 0.1 in these spectra) — 1e-4 absolute covers it with margin.  Flags are
compared only where no oracle angle lies within a factor 2 of tol (a floating-point-decided integer).
"""
import math

import numpy as np
import pytest

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


def _planted(n, d, seed):
    """exponential spectrum 100 → 0.1 with a Haar basis (P L365's synthetic family), fp32"""
    rng = np.random.default_rng(seed)
    lam = 100.0 * (1e-3) ** (np.arange(d) / (d - 1))
    q, r = np.linalg.qr(rng.standard_normal((d, d)))
    q *= np.sign(np.diag(r))
    return ((rng.standard_normal((n, d)) * np.sqrt(lam)) @ q.T).astype(np.float32)


def _run(P, ctx, X, V, T, upto, tol):
    import torch
    Xd = U.upload(X, "f32")
    Xm = P.matrix(Xd, d=X.shape[1])
    Vd = torch.from_numpy(np.ascontiguousarray(V, dtype=np.float32)).cuda()
    Td = torch.from_numpy(np.ascontiguousarray(T[:upto], dtype=np.float32)).cuda()
    return P.ppca_check_prop3(ctx, Xm, Vd, V.shape[0], Td, upto, tol)


def _compare(flags_d, ang_d, X, V, T, upto, tol, atol):
    flags_o, ang_o = O.check_prop3(X.astype(np.float64), V.astype(np.float64), T.astype(np.float64), upto, tol)
    np.testing.assert_allclose(ang_d, ang_o, atol=atol, rtol=1e-3)
    # chain semantics on the device's own angles
    chain = True
    for i in range(upto):
        chain = chain and ang_d[i] <= tol
        assert flags_d[i] == chain
    if all(abs(math.log(max(a, 1e-300) / tol)) > math.log(2) for a in ang_o):
        assert flags_d == flags_o
    return ang_o


@pytest.mark.parametrize("n,d,k,extra,noise,tol", [(3000, 40, 6, 2, 0.05, 1e-2), (3000, 40, 6, 2, 0.5, 1e-2),
                                                   (2500, 96, 10, 70, 0.02, 1e-2)])
def test_prop3_parity_random_priming(P, ctx, n, d, k, extra, noise, tol):
    X = _planted(n, d, 50 + d)
    _, T = O.truth(X.astype(np.float64))
    T = T.astype(np.float32)
    rng = np.random.default_rng(51)
    V = np.vstack([T[:k] + noise * rng.standard_normal((k, d)), rng.standard_normal((extra, d))]).astype(np.float32)
    flags, ang = _run(P, ctx, X, V, T, k, tol)
    _compare(flags, ang, X, V, T, k, tol, 1e-4)


def test_prop3_truth_holds_on_gpu(P, ctx):
    X = _planted(2000, 32, 60)
    _, T = O.truth(X.astype(np.float64))
    T = T.astype(np.float32)
    flags, ang = _run(P, ctx, X, T[:5], T, 5, 1e-4)
    assert all(flags) and np.all(ang < 1e-5)


def test_prop3_paper_counterexample_on_gpu(P, ctx):
    """§4.1 (P L195–223), ε = 0.01: condition 1 fails at angle π/2 (S L346)."""
    eps = 0.01
    X = np.array([[3, 0, 0], [-3, 0, 0], [0, 2, 0], [0, -2, 0], [0, 0, 1], [0, 0, -1]], dtype=np.float32)
    V = np.array([[eps, 0, math.sqrt(1 - eps ** 2)], [0, 1, 0]], dtype=np.float32)
    flags, ang = _run(P, ctx, X, V, np.eye(3, dtype=np.float32), 2, 1e-8)
    assert flags == [False, False]
    assert ang[0] == pytest.approx(math.pi / 2, abs=1e-6)


@pytest.mark.parametrize("delta2,expect_flags,expect_ang", [
    (0.6, [True, True, True], [0, 0, 0]),
    (0.8, [True, False, False], [0, math.pi / 2, 0])])
def test_prop3_closed_form_on_gpu(P, ctx, delta2, expect_flags, expect_ang):
    """XᵀX = diag(10, 6, 4, 2, 1, ½), S = span(e1, e2 + δe5, e3): condition 2 holds iff δ² < 2/3 (the
    oracle pin test_prop3_closed_form_condition2_and_chain); the chain breaks at the first failure."""
    X = np.diag(np.sqrt([10, 6, 4, 2, 1, 0.5])).astype(np.float32)
    dd = math.sqrt(delta2)
    V = np.array([[1, 0, 0, 0, 0, 0], [0, 1, 0, 0, dd, 0], [0, 0, 1, 0, 0, 0]], dtype=np.float32)
    flags, ang = _run(P, ctx, X, V, np.eye(6, dtype=np.float32), 3, 1e-5)
    assert flags == expect_flags
    np.testing.assert_allclose(ang, expect_ang, atol=1e-6)


def test_prop3_errors(P, ctx):
    X = np.diag(np.sqrt([5, 3, 2, 1])).astype(np.float32)
    V = np.array([[0, 1, 0, 0], [0, 0, 1, 0]], dtype=np.float32)
    with pytest.raises(P.PPCAError) as ei:                   # π_S(e1) = 0 (S L343)
        _run(P, ctx, X, V, np.eye(4, dtype=np.float32), 2, 1e-8)
    assert ei.value.name == "PPCA_ERR_DEGENERATE"
    with pytest.raises(P.PPCAError) as ei:                   # dim S = 2 < upto = 3
        _run(P, ctx, X, V, np.eye(4, dtype=np.float32), 3, 1e-8)
    assert ei.value.name == "PPCA_ERR_SUBSPACE_COLLAPSE"
