"""More pins of the fp64 oracle (no GPU): the subspace error (C5's target metric, reading R20), the power
method's stop rule (P L61-62) and the residual-certified reference (reading R29).

Each test fixes the function against a closed form, a textbook bound or an independent library routine,
so a dropped term, a transposed projector, a wrong sign or an off-by-one stop fails."""
import math

import numpy as np
import pytest
import scipy.linalg

from oracle import ppca_oracle as O


# ----------------------------------------------------------------------------- subspace error (R20)
@pytest.mark.parametrize("angles", [[0.0, 0.0, 0.0], [0.1, 0.02, 0.3], [math.pi / 2, 0.0, 0.01]])
def test_subspace_error_closed_form_principal_angles(angles):
    """E_i = cos a_i e_i + sin a_i e_{k+i}, T_i = e_i: the principal angles are exactly a_i, so the error is
    max sin a_i — for any rotation of T within its span and any ordering of E's rows."""
    k, d = len(angles), 9
    T = np.eye(d)[:k]
    E = np.array([math.cos(a) * np.eye(d)[i] + math.sin(a) * np.eye(d)[k + i] for i, a in enumerate(angles)])
    want = max(math.sin(a) for a in angles)
    assert O.subspace_error(E, T) == pytest.approx(want, abs=1e-15)
    rng = np.random.default_rng(3)
    Q = np.linalg.qr(rng.standard_normal((k, k)))[0]
    assert O.subspace_error(E, Q @ T) == pytest.approx(want, abs=1e-14)          # basis of span T
    assert O.subspace_error(E[::-1], T) == pytest.approx(want, abs=1e-14)        # order of E's rows
    # independent routine: scipy's principal angles (column bases)
    assert O.subspace_error(E, T) == pytest.approx(math.sin(np.max(scipy.linalg.subspace_angles(E.T, T.T))),
                                                   abs=1e-12)


def test_subspace_error_generic_vs_scipy_and_not_transposed():
    """Random k-dim subspaces of R^d with d > 2k: against scipy's principal angles.  A projector built from
    E instead of T, or a transposed product, gives a different value on this non-symmetric configuration."""
    rng = np.random.default_rng(11)
    d, k = 30, 4
    T = np.linalg.qr(rng.standard_normal((d, k)))[0].T
    E = np.linalg.qr((T.T + 0.3 * rng.standard_normal((d, k))))[0].T
    ref = math.sin(np.max(scipy.linalg.subspace_angles(E.T, T.T)))
    assert O.subspace_error(E, T) == pytest.approx(ref, rel=1e-12)
    assert 0.05 < ref < 0.99


# ----------------------------------------------------------------------------- power stop rule (P L61-62)
def test_power_stop_rule_closed_form():
    """One vector on M = diag(λ1, λ2): w_t = (cos φ_t, sin φ_t) with tan φ_t = (λ2/λ1)^t tan φ_0 (P L61), so
    ‖w_{t+1} − w_t‖ = 2 sin((φ_t − φ_{t+1})/2); the method stops after the first step whose move is < ε."""
    lam = np.array([4.0, 1.0])
    X = np.diag(np.sqrt(lam))                      # XᵀX = diag(λ)
    W0 = np.array([[1.0, 2.0]])
    phi0 = math.atan2(2.0, 1.0)
    for eps in [0.3, 1e-2, 1e-5]:
        t, phi = 0, phi0
        while True:
            nxt = math.atan((lam[1] / lam[0]) ** (t + 1) * math.tan(phi0))
            t += 1
            move = 2 * math.sin((phi - nxt) / 2)
            phi = nxt
            if move < eps:
                break
        W, S_hist = O.prime_power(X, W0, 100, eps=eps)
        assert len(S_hist) == t, f"eps={eps}: oracle stopped after {len(S_hist)}, closed form {t}"
        assert W[0] @ np.array([math.cos(phi), math.sin(phi)]) == pytest.approx(1.0, abs=1e-12)
    # eps = 0: the full budget
    _, S_hist = O.prime_power(X, W0, 17)
    assert len(S_hist) == 17


def test_column_moves_sign_invariant():
    w = np.array([[0.6, 0.8, 0.0]])
    assert O.column_moves(-w, w)[0] == 0.0
    assert O.column_moves(np.array([[0.0, 0.0, 1.0]]), w)[0] == pytest.approx(math.sqrt(2.0))


# ----------------------------------------------------------------------------- certified reference (O9, R29)
def _planted(n, d, lam, seed):
    rng = np.random.default_rng(seed)
    Q = np.linalg.qr(rng.standard_normal((d, d)))[0]
    X = rng.standard_normal((n, d)) * np.sqrt(lam) @ Q.T
    return X - X.mean(axis=0)


def test_certified_top_bounds_hold_against_exact_eigensystem():
    """Weyl: every certified θ_i has a true eigenvalue within r_i; Davis–Kahan: the true angle of e_i is below
    r_i/gap_i and the true top-k subspace error below ‖R_k‖/δ — checked against the exact eigensystem of
    the formed XᵀX (LAPACK), on a spectrum with gaps."""
    n, d, k, m = 600, 48, 5, 10
    lam = np.exp(-np.arange(1, d + 1) / 4.0)
    X = _planted(n, d, lam, 5)
    ev, T = O.truth(X)
    rng = np.random.default_rng(8)
    # stopped early (loose residuals): the bounds must still hold and be non-trivial
    for iters, rtol in [(6, 0.0), (500, 1e-11)]:
        c = O.certified_top(X, k, rng.standard_normal((m, d)), max_iters=iters, rtol=rtol)
        th, E, res = c["theta"], c["E"], c["res"]
        for i in range(k):
            assert np.min(np.abs(ev - th[i])) <= res[i] * (1 + 1e-9) + 1e-12 * ev[0]      # Weyl
            sin = np.linalg.norm(E[i] - (E[i] @ T[i]) * T[i])                             # accurate at tiny angles
            assert sin <= c["angle_bound"][i] * (1 + 1e-9) + 1e-12                        # Davis–Kahan
        assert O.subspace_error(E, T[:k]) <= c["subspace_bound"] * (1 + 1e-9) + 1e-12    # sinΘ
        assert np.all(th <= ev[:k] * (1 + 1e-12))                                         # Cauchy interlacing
    # converged: θ equal to the eigenvalues, bounds tiny
    assert c["iters"] < 500
    np.testing.assert_allclose(th, ev[:k], rtol=1e-10)
    assert c["subspace_bound"] < 1e-8 and np.max(c["angle_bound"]) < 1e-8


def test_certified_top_residual_is_the_eigen_residual():
    """The residual of an exact eigenvector is zero, and of a perturbed one equals ‖(M − θ)e‖ (a certifier
    that used the wrong θ order or a transposed product would report a large residual at convergence)."""
    n, d, k, m = 300, 20, 3, 6
    lam = 1.0 / np.arange(1, d + 1)
    X = _planted(n, d, lam, 2)
    M = X.T @ X
    c = O.certified_top(X, k, np.random.default_rng(1).standard_normal((m, d)), max_iters=2000, rtol=1e-12)
    for i in range(k):
        e = c["E"][i]
        assert np.linalg.norm(M @ e - c["theta"][i] * e) <= 1e-11 * c["theta"][0] + c["res"][i] * 1.01
    assert np.all(c["res"] <= 1e-12 * c["theta"][0] * 1.0001)


def test_ritz_residuals_closed_form():
    """M = diag(λ1, λ2) (X = diag(√λ)), e = (cos a, sin a), θ = its Rayleigh quotient:
    Me − θe = (λ1 − λ2) sin a cos a (sin a, −cos a), so r = (λ1 − λ2)|sin a cos a|; r = 0 at an eigenvector."""
    lam = np.array([5.0, 2.0])
    X = np.diag(np.sqrt(lam))
    for a in [0.0, 0.1, 0.7]:
        e = np.array([[math.cos(a), math.sin(a)]])
        th = lam[0] * math.cos(a) ** 2 + lam[1] * math.sin(a) ** 2
        r = O.ritz_residuals(X, e, [th])[0]
        assert r == pytest.approx((lam[0] - lam[1]) * abs(math.sin(a) * math.cos(a)), abs=1e-14)
    # a wrong θ shows up in full: ‖(M − θ')e‖ at an exact eigenvector
    assert O.ritz_residuals(X, np.array([[1.0, 0.0]]), [4.0])[0] == pytest.approx(1.0, abs=1e-14)


# ----------------------------------------------------------------------------- Theorem 1 (NEXT-4)
def test_theorem1_counterexample_conditions_fail_and_conclusion_fails():
    """§4.1 (P L195-228): condition 1 fails (upto = 0), and indeed pPCA's first vector (e2) is farther from e1
    than the priming's first vector — the theorem's conclusion needs its conditions (the check is not vacuous)."""
    X = np.array([[3, 0, 0], [-3, 0, 0], [0, 2, 0], [0, -2, 0], [0, 0, 1], [0, 0, -1]], dtype=float)
    eps = 0.01
    V = np.array([[eps, 0, math.sqrt(1 - eps ** 2)], [0, 1, 0]])
    lam, T = O.truth(X)
    upto, a_prim, a_ppca, holds = O.theorem1_check(X, V, T, 2, tol=1e-8)
    assert upto == 0 and holds                       # vacuously true on an empty run …
    assert a_ppca[0] > a_prim[0]                     # … and the conclusion indeed fails without condition 1


def test_theorem1_holds_whenever_conditions_hold():
    """Near-converged primings (V = T + δ·noise, the regime Theorem 1 describes): conditions hold on a run and
    the pPCA angles never exceed the priming's there; larger δ shortens the run."""
    rng = np.random.default_rng(4)
    n, d, k, l = 800, 30, 6, 4
    lam = np.exp(-np.arange(1, d + 1) / 3.0)
    Q = np.linalg.qr(rng.standard_normal((d, d)))[0]
    X = rng.standard_normal((n, d)) * np.sqrt(lam) @ Q.T
    X -= X.mean(axis=0)
    _, T = O.truth(X)
    runs = []
    for delta in [1e-4, 1e-3, 1e-2, 5e-2]:
        for seed in range(3):
            noise = np.random.default_rng(seed).standard_normal((k + l, d))
            V = np.vstack([T[: k + l]]) + delta * noise
            upto, a_prim, a_ppca, holds = O.theorem1_check(X, V, T, k, tol=1e-6)
            assert holds, (delta, seed, upto)
            runs.append(upto)
            if upto == k:
                lp = [O.lces(a_prim, v) for v in O.PI_THRESHOLDS]
                lq = [O.lces(a_ppca, v) for v in O.PI_THRESHOLDS]
                assert all(q >= p for p, q in zip(lp, lq))
    assert runs[0] == k                              # the smallest perturbation: all k conditions hold
