"""Pins of the fp64 oracle against what the paper and the mathematics fix (no GPU).

Each test names the passage it pins.  A plausible slip in the oracle (dropped term,
wrong sign, transposed operand, wrong triangle, mean instead of sum, missing
tangent projection, wrong Nesterov form, off-by-one streak) fails at least one.
"""
import math
import os

import numpy as np
import pytest

from oracle import ppca_oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _read_kv(name):
    out = {}
    with open(os.path.join(GOLD, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            k, v = line.split(":", 1)
            out[k.strip()] = v.strip()
    return out


def _counterexample():
    g = _read_kv("counterexample_4_1.txt")
    pts = [list(map(float, p.split())) for p in g["points"].split("|")]
    return np.array(pts), g


# ----------------------------------------------------------------------------- §4.1 counterexample (T1)
def test_counterexample_covariance_and_order_swap():
    X, g = _counterexample()
    eps = float(g["eps"])
    cov = O.covariance(X, normalize=True)
    np.testing.assert_allclose(np.diag(cov), list(map(float, g["cov_normalized_diag"].split())), atol=1e-15)
    assert np.count_nonzero(cov - np.diag(np.diag(cov))) == 0
    # truth e1=(1,0,0), e2=(0,1,0)  (P L204)
    lam, T = O.truth(X)
    np.testing.assert_allclose(T[0], [1, 0, 0], atol=1e-15)
    np.testing.assert_allclose(T[1], [0, 1, 0], atol=1e-15)
    # priming output (P L206) and projected covariance (corrected P L218, reading R22)
    P = np.array([[eps, 0.0, math.sqrt(1 - eps ** 2)], [0.0, 1.0, 0.0]])
    B = O.gram_schmidt(P)
    S = O.projected_gram(X, B) / X.shape[0]
    np.testing.assert_allclose(np.diag(S), list(map(float, g["projected_cov_normalized_diag"].split())), rtol=1e-14)
    assert abs(S[0, 1]) < 1e-15
    # pPCA swaps the order (P L222-227)
    E, theta, _, _ = O.ppca_refine(X, P, k=2)
    np.testing.assert_allclose(E[0], list(map(float, g["ppca_e1"].split())), atol=1e-14)
    np.testing.assert_allclose(E[1], list(map(float, g["ppca_e2"].split())), atol=1e-14)
    assert abs(E[0] @ T[0]) ** 2 == 0.0
    assert abs(P[0] @ T[0]) ** 2 == pytest.approx(eps ** 2, rel=1e-12)
    assert O.captured_variance(X, np.array([1.0, 0, 0])) == float(g["captured_variance_e1"])


# ----------------------------------------------------------------------------- LCES (T2)
def test_lces_worked_example_and_monotone():
    g = _read_kv("lces_worked_example.txt")
    ratios = list(map(float, g["angles_over_V"].split()))
    for V in O.PI_THRESHOLDS:
        assert O.lces([r * V for r in ratios], V) == int(g["lces"])
    rng = np.random.default_rng(0)
    for _ in range(200):
        a = rng.uniform(0, 0.5, size=8)
        s = [O.lces(a, V) for V in O.PI_THRESHOLDS]
        assert all(s[i] >= s[i + 1] for i in range(len(s) - 1))
    assert O.lces([0.0] * 5, 0.1) == 5
    assert O.lces([0.2, 0.0], 0.1) == 0
    assert O.lces([0.1], 0.1) == 0                      # strict "<" (P L412 "smaller than V")
    assert O.angular_error(np.array([1.0, 0]), np.array([-1.0, 0])) == 0.0
    assert O.angular_error(np.array([1.0, 0]), np.array([0, 1.0])) == pytest.approx(math.pi / 2)


# ----------------------------------------------------------------------------- Jacobi (T3)
def test_jacobi_analytic_and_lapack():
    vals, vecs = O.jacobi_eigh(np.array([[2.0, 1.0], [1.0, 2.0]]))
    np.testing.assert_allclose(vals, [3.0, 1.0], atol=1e-15)
    np.testing.assert_allclose(np.abs(vecs), np.full((2, 2), 1 / math.sqrt(2)), atol=1e-15)
    vals, vecs = O.jacobi_eigh(np.diag([9.0, 4.0, 1.0]) / 3)
    np.testing.assert_allclose(vals, [3, 4 / 3, 1 / 3], atol=1e-15)
    np.testing.assert_allclose(vecs, np.eye(3), atol=0)
    rng = np.random.default_rng(1)
    for n in (3, 8, 17, 40):
        A = rng.standard_normal((n, n))
        A = A + A.T
        vals, vecs = O.jacobi_eigh(A)
        ref = np.sort(np.linalg.eigvalsh(A))[::-1]
        np.testing.assert_allclose(vals, ref, rtol=0, atol=1e-12 * np.abs(ref).max())
        recon = vecs.T @ np.diag(vals) @ vecs
        assert np.linalg.norm(recon - A) < 1e-12 * np.linalg.norm(A)
        np.testing.assert_allclose(vecs @ vecs.T, np.eye(n), atol=1e-13)
        # eigenvectors: each row satisfies A v = λ v
        for i in range(n):
            assert np.linalg.norm(A @ vecs[i] - vals[i] * vecs[i]) < 1e-11 * np.abs(vals).max()
        # sign convention
        for i in range(n):
            j = int(np.argmax(np.abs(vecs[i])))
            assert vecs[i, j] > 0


def test_jacobi_tie_order_is_stable():
    vals, vecs = O.jacobi_eigh(np.diag([1.0, 2.0, 2.0]))
    np.testing.assert_allclose(vals, [2, 2, 1])
    np.testing.assert_allclose(vecs, [[0, 1, 0], [0, 0, 1], [1, 0, 0]])


# ----------------------------------------------------------------------------- Gram–Schmidt (T4)
def test_gram_schmidt_examples():
    B = O.gram_schmidt(np.array([[2.0, 0, 0], [1.0, 1.0, 0]]))
    np.testing.assert_allclose(B, [[1, 0, 0], [0, 1, 0]], atol=1e-15)
    B = O.gram_schmidt(np.array([[1.0, 0, 0], [1.0, 1e-13, 0]]))
    assert B.shape == (1, 3)
    with pytest.raises(O.SubspaceCollapse):
        O.gram_schmidt(np.array([[1.0, 0, 0], [1.0, 1e-13, 0]]), drop=False)
    rng = np.random.default_rng(2)
    V = rng.standard_normal((7, 30))
    B = O.gram_schmidt(V)
    np.testing.assert_allclose(B @ B.T, np.eye(7), atol=1e-14)
    np.testing.assert_allclose(O.gram_schmidt(B), B, atol=1e-12)          # idempotent
    # same Q as a Householder QR with positive diag(R)
    q, r = np.linalg.qr(V.T)
    q = q * np.sign(np.diag(r))[None, :]
    np.testing.assert_allclose(B, q.T, atol=1e-13)


# ----------------------------------------------------------------------------- EigenGame utilities (T5)
def test_eigengame_utilities_values():
    M = np.diag([3.0, 2.0, 1.0])
    np.testing.assert_allclose(O.eigengame_utilities(M, np.eye(3)[:2]), [3.0, 2.0], atol=0)
    v = np.array([0.6, 0.8, 0.0])
    assert O.eigengame_utilities(M, np.stack([v, v]))[1] == pytest.approx(0.0, abs=1e-15)
    M = np.diag([2.0, 1.0])
    V = np.array([[1, 1], [1, -1]]) / math.sqrt(2)
    np.testing.assert_allclose(O.eigengame_utilities(M, V), [1.5, 4 / 3], atol=1e-12)
    # even in each vector
    np.testing.assert_allclose(O.eigengame_utilities(M, V * np.array([[-1], [1]])), [1.5, 4 / 3], atol=1e-12)


def test_eigengame_step_hand_values():
    # X with XᵀX = diag(2,1); V = [(1,1)/√2, (1,-1)/√2]; hand-derived (DESIGN.md §Oracle pins):
    # ∇_1 = 2Mv_1 = √2(2,1), <∇_1,v_1> = 3 ⇒ r_1 = (1,-1)/√2 ;  ∇_2 = 2Mv_2 − (2/3)Mv_1 ⇒ r_2 = 0.
    X = np.array([[math.sqrt(2), 0.0], [0.0, 1.0]])
    V = np.array([[1.0, 1.0], [1.0, -1.0]]) / math.sqrt(2)
    alpha = 0.1
    Vn, vel = O.eigengame_step(X, V, np.zeros_like(V), alpha, 0.0)
    r1 = np.array([1.0, -1.0]) / math.sqrt(2)
    np.testing.assert_allclose(vel[0], r1, atol=1e-14)
    np.testing.assert_allclose(vel[1], [0, 0], atol=1e-14)
    exp1 = V[0] + alpha * r1
    np.testing.assert_allclose(Vn[0], exp1 / np.linalg.norm(exp1), atol=1e-14)
    np.testing.assert_allclose(Vn[1], V[1], atol=1e-14)
    # tangent identity <∇_j, v_j> = 2 U_j (P Eq. 3)
    U = O.eigengame_utilities(X.T @ X, V)
    np.testing.assert_allclose(U, [1.5, 4 / 3], atol=1e-12)


# ----------------------------------------------------------------------------- Oja single steps
def test_oja_hand_values_sum_and_triangle():
    # m=1: x=(1,0), w=(1,1): y=1, G = yx − y²w = (0,-1); α=0.1, μ=0 ⇒ w'=(1, 0.9)  (P L67)
    W, vel = O.oja_step(np.array([[1.0, 0.0]]), np.array([[1.0, 1.0]]), np.zeros((1, 2)), 0.1, 0.0)
    np.testing.assert_allclose(W, [[1.0, 0.9]], atol=1e-15)
    # m=2 Sanger (P L71, Σ_{l≤m}): w1=e1, w2=e2, x=(1,1): G1 = (0,1), G2 = (0,0)
    W0 = np.eye(2)
    W, vel = O.oja_step(np.array([[1.0, 1.0]]), W0, np.zeros((2, 2)), 1.0, 0.0)
    np.testing.assert_allclose(vel, [[0, 1], [0, 0]], atol=1e-15)
    # batch SUM, not mean (reading R8): two identical rows double the step
    W1, v1 = O.oja_step(np.array([[1.0, 1.0]]), W0, np.zeros((2, 2)), 1.0, 0.0)
    W2, v2 = O.oja_step(np.array([[1.0, 1.0], [1.0, 1.0]]), W0, np.zeros((2, 2)), 1.0, 0.0)
    np.testing.assert_allclose(v2, 2 * v1, atol=1e-15)
    # α = 0 no-op (S L237)
    rng = np.random.default_rng(3)
    Wr = rng.standard_normal((3, 5))
    Wn, _ = O.oja_step(rng.standard_normal((4, 5)), Wr, np.zeros((3, 5)), 0.0, 0.9)
    np.testing.assert_array_equal(Wn, Wr)


# ----------------------------------------------------------------------------- fixed points (T6)
def _random_data(n, d, seed):
    rng = np.random.default_rng(seed)
    lam = np.exp(-np.arange(d) / 2.0)
    q, _ = np.linalg.qr(rng.standard_normal((d, d)))
    return (rng.standard_normal((n, d)) * np.sqrt(lam)) @ q.T


def _moved(A, B):
    """max over rows of the sign-aligned distance ‖a − sign(a·b) b‖ (≈ angle for tiny angles;
    arccos of a cosine near 1 cannot resolve angles below ~1e-8)."""
    return max(np.linalg.norm(a / np.linalg.norm(a) - np.sign(a @ b) * b) for a, b in zip(A, B))


def test_fixed_points_full_batch():
    X = _random_data(500, 10, 4)
    lam, T = O.truth(X)
    Wt = T[:3]
    W1, _ = O.power_step(X, Wt)
    assert _moved(W1, Wt) < 1e-9
    # Oja: w = exact unit eigenvector ⇒ G = Cw − (wᵀCw)w = 0 for m=1 (P L69)
    Wo, _ = O.oja_step(X, Wt[:1], np.zeros((1, 10)), 1e-3, 0.9)
    assert _moved(Wo, Wt[:1]) < 1e-9
    # Sanger with m=3 exact eigenvectors: also a fixed point
    Wo, _ = O.oja_step(X, Wt, np.zeros((3, 10)), 1e-4, 0.0)
    assert _moved(Wo, Wt) < 1e-9
    Ve, _ = O.eigengame_step(X, Wt, np.zeros((3, 10)), 1e-3, 0.9)
    assert _moved(Ve, Wt) < 1e-9


# ----------------------------------------------------------------------------- power contraction (T7)
def test_power_contraction_rate_closed_form():
    X = np.array([[math.sqrt(2.0), 0.0], [0.0, 1.0]])         # XᵀX = diag(2,1)
    W = np.array([[1.0, 1.0]]) / math.sqrt(2)
    prev = 1.0                                                 # tan θ_0 = 1
    for t in range(20):
        W, _ = O.power_step(X, W)
        tan = abs(W[0, 1] / W[0, 0])
        assert tan / prev == pytest.approx(0.5, abs=1e-6)      # (λ2/λ1)^t tan θ_0
        prev = tan


# ----------------------------------------------------------------------------- Nesterov (T8)
def test_nesterov_unroll():
    p, v = O.nesterov_update(np.zeros(2), np.zeros(2), np.ones(2), 1.0, 0.0)
    np.testing.assert_allclose(p, [1, 1])
    p, v = O.nesterov_update(np.zeros(2), np.zeros(2), np.zeros(2), 0.5, 0.9)
    np.testing.assert_allclose(p, [0, 0])
    g = np.array([1.0, -2.0])
    p, v = O.nesterov_update(np.zeros(2), np.zeros(2), g, 1.0, 0.9)
    np.testing.assert_allclose(p, g * 1.9)
    p, v = O.nesterov_update(p, v, g, 1.0, 0.9)
    np.testing.assert_allclose(p, g * 1.9 + g * (1 + 0.9 + 0.81))


# ----------------------------------------------------------------------------- Oja ascent (T9)
def test_oja_rayleigh_non_decreasing():
    X = _random_data(400, 10, 5)
    C = X.T @ X
    rng = np.random.default_rng(6)
    w = rng.standard_normal((1, 10))
    vel = np.zeros_like(w)
    alpha = 1e-3 / np.linalg.eigvalsh(C)[-1]
    rq = lambda w: float(w[0] @ C @ w[0] / (w[0] @ w[0]))
    prev = rq(w)
    for _ in range(100):
        w, vel = O.oja_step(X, w, vel, alpha, 0.0)
        cur = rq(w)
        assert cur >= prev - 1e-12 * abs(prev)
        prev = cur


# ----------------------------------------------------------------------------- pPCA invariants (T10, T11)
def test_ppca_invariants():
    X = _random_data(300, 12, 7)
    lam, T = O.truth(X)
    d = X.shape[1]
    rng = np.random.default_rng(8)
    # (a) full orthonormal basis ⇒ exact PCA
    Q, _ = np.linalg.qr(rng.standard_normal((d, d)))
    E, th, _, _ = O.ppca_refine(X, Q.T, k=d)
    assert max(O.angles(E, T)) < 1e-8
    np.testing.assert_allclose(th, lam, rtol=1e-11)
    # brute force: pPCA on the full space equals Jacobi of XᵀX itself
    vals_bf, vecs_bf = O.jacobi_eigh(X.T @ X)
    np.testing.assert_allclose(th, vals_bf, rtol=1e-11)
    # primed = random rotation of the top-4 span (l=0) ⇒ exact top-4
    R, _ = np.linalg.qr(rng.standard_normal((4, 4)))
    E, th, _, _ = O.ppca_refine(X, R @ T[:4], k=4)
    assert max(O.angles(E, T[:4])) < 1e-10
    np.testing.assert_allclose(th, lam[:4], rtol=1e-12)
    # (e) exact eigenvectors ⇒ identity
    E, th, _, _ = O.ppca_refine(X, T[:5], k=5)
    np.testing.assert_allclose(E, T[:5], atol=1e-12)
    # random m-dim priming
    V = T[:6] + 0.3 * rng.standard_normal((6, d))
    E, th, th_all, _ = O.ppca_refine(X, V, k=3)
    # (b) span only: permutation + sign flips
    E2, th2, _, _ = O.ppca_refine(X, -V[::-1], k=3)
    np.testing.assert_allclose(E2, E, atol=1e-12)
    np.testing.assert_allclose(th2, th, rtol=1e-12)
    # (f) idempotent
    E3, th3, _, _ = O.ppca_refine(X, E, k=3)
    np.testing.assert_allclose(E3, E, atol=1e-12)
    # (d) Cauchy interlacing λ_{i+d−m} ≤ θ_i ≤ λ_i
    m = 6
    for i in range(m):
        assert lam[i + d - m] - 1e-9 <= th_all[i] <= lam[i] + 1e-9
    # (c) Rayleigh quotients of the orthonormalised priming vs pPCA: θ_1 ≥ max ρ, Ky Fan sums
    B = O.gram_schmidt(V)
    rho = np.sort([b @ X.T @ X @ b for b in B])[::-1]
    assert th_all[0] >= rho[0] - 1e-9
    for j in range(m):
        assert th_all[: j + 1].sum() >= rho[: j + 1].sum() - 1e-9 * abs(rho).sum()
    # the captured variance of each Ritz vector equals its Ritz value
    for i in range(3):
        assert O.captured_variance(X, E[i]) == pytest.approx(th[i], rel=1e-12)


def test_ppca_subspace_collapse():
    X = _random_data(50, 5, 9)
    V = np.array([[1.0, 0, 0, 0, 0], [2.0, 0, 0, 0, 0]])
    with pytest.raises(O.SubspaceCollapse):
        O.ppca_refine(X, V, k=2)


def test_theorem1_mechanism_near_converged():
    """Prop. 3 / Thm 1 (P L293–321): once the primed vectors are close to the truth, the
    full-PCA step does not shorten the streak at any V (tested as the non-strict inequality)."""
    X = _random_data(2000, 10, 10)
    lam, T = O.truth(X)
    rng = np.random.default_rng(11)
    for trial in range(20):
        V = T[:4] + 1e-3 * rng.standard_normal((4, 10))
        V = O.normalize_rows(V)
        E, _, _, _ = O.ppca_refine(X, V, k=4)
        a_prime, a_ppca = O.angles(V, T[:4]), O.angles(E, T[:4])
        for thr in O.PI_THRESHOLDS:
            assert O.lces(a_ppca, thr) >= O.lces(a_prime, thr)


def test_relative_gaps():
    g = O.relative_gaps(np.array([10.0, 5.0, 4.0, 1.0]))
    np.testing.assert_allclose(g, [0.5, 0.2, 0.25, 3.0])


# ----------------------------------------------------------------------------- row-subsampled refine (R25)
def test_sampled_refine_reduces_to_refine_and_is_unbiased():
    X = _random_data(3000, 10, 21)
    rng = np.random.default_rng(22)
    V = rng.standard_normal((6, 10))
    # fraction 1 is the plain refine
    E1, th1, used = O.ppca_refine_sampled(X, V, 3, 1.0, 5)
    E0, th0, _, _ = O.ppca_refine(X, V, 3)
    assert used == 3000
    np.testing.assert_allclose(th1, th0, rtol=1e-13)
    np.testing.assert_allclose(E1, E0, atol=1e-12)
    # the sample is whole 128-row tiles, deterministic in the seed, about `fraction` of them
    rows = O.sampled_rows(100_000, 0.1, 7)
    cnt = np.bincount(rows // 128, minlength=782)          # 100000 rows = 781 full tiles + 32
    assert np.all(np.isin(cnt[:-1], [0, 128])) and cnt[-1] in (0, 32)
    np.testing.assert_array_equal(rows, O.sampled_rows(100_000, 0.1, 7))
    assert abs(rows.size / 100_000 - 0.1) < 0.02
    # the rescaled projected covariance is an unbiased estimate: mean over seeds ≈ the full one
    B = O.gram_schmidt(V)
    S_full = O.projected_gram(X, B)
    acc = np.zeros_like(S_full)
    seeds = range(40)
    for sd in seeds:
        r = O.sampled_rows(3000, 0.5, sd)
        acc += O.projected_gram(X[r], B) * (3000 / r.size)
    acc /= len(seeds)
    assert np.linalg.norm(acc - S_full) / np.linalg.norm(S_full) < 0.05


# ----------------------------------------------------------------------------- Prop. 3 checker (NEXT-4)
def _diag_data(lam):
    """rows √λ_j e_j: XᵀX = diag(λ) exactly, the true eigenvectors are the unit vectors"""
    return np.diag(np.sqrt(np.asarray(lam, dtype=np.float64)))


def test_prop3_truth_and_containing_span_hold():
    """S L341/L346 [TRIVIAL]: primed = truth → π_S(e_i) = e_i, every condition holds; a primed set whose span
    contains the top-k truth (rotated, plus extra random directions) holds for i ≤ k as well."""
    X = _random_data(2000, 10, 31)
    lam, T = O.truth(X)
    flags, ang = O.check_prop3(X, T[:4], T, 4)
    assert all(flags) and np.all(ang < 1e-12)
    rng = np.random.default_rng(32)
    Q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
    V = np.vstack([Q @ T[:3], rng.standard_normal((2, 10))])
    flags, ang = O.check_prop3(X, V, T, 3)
    assert all(flags) and np.all(ang < 1e-9)


def test_prop3_paper_counterexample():
    """§4.1 (P L195–223): X = {±3e1, ±2e2, ±e3}, priming (ε, 0, √(1−ε²)), (0, 1, 0), ε = 0.01.  Projected
    variance along e_1^priming is 2(9ε² + (1−ε²)) < 8 (reading R22), so the top direction of the projected
    data is e_2 and π_S(e_1) ∝ e_1^priming is orthogonal to it: condition 1 fails at angle π/2
    (S L346 "flag[1] = false"); the pPCA output is (0, 1, 0) first (P L219–222)."""
    eps = 0.01
    X = np.array([[3, 0, 0], [-3, 0, 0], [0, 2, 0], [0, -2, 0], [0, 0, 1], [0, 0, -1]], dtype=np.float64)
    V = np.array([[eps, 0, math.sqrt(1 - eps ** 2)], [0, 1, 0]])
    T = np.eye(3)
    flags, ang = O.check_prop3(X, V, T, 2)
    assert flags == [False, False]
    assert ang[0] == pytest.approx(math.pi / 2, abs=1e-12)
    E, _, _, _ = O.ppca_refine(X, V, 2)
    np.testing.assert_allclose(np.abs(E[0]), [0, 1, 0], atol=1e-12)


@pytest.mark.parametrize("delta2,expect", [(0.7, [True, True, True]), (0.9, [False, False, False])])
def test_prop3_closed_form_threshold_condition1(delta2, expect):
    """Closed form: XᵀX = diag(λ), S = span(e1 + δe5, e2, e3).  In the basis {f ∝ e1 + δe5, e2, e3} the
    projected covariance is diagonal with Var(f) = (λ1 + δ²λ5)/(1 + δ²), and π_S(e1) ∝ f.  Condition 1
    holds iff Var(f) > λ2 ⟺ δ² < (λ1 − λ2)/(λ2 − λ5) = 0.8 for λ = (10, 6, 4, 2, 1, ½); when it fails,
    the maximiser is e2 ⊥ f: angle π/2."""
    lam = [10, 6, 4, 2, 1, 0.5]
    X = _diag_data(lam)
    d = math.sqrt(delta2)
    V = np.array([[1, 0, 0, 0, d, 0], [0, 1, 0, 0, 0, 0], [0, 0, 1, 0, 0, 0]], dtype=np.float64)
    flags, ang = O.check_prop3(X, V, np.eye(6), 3)
    assert flags == expect
    np.testing.assert_allclose(ang, [0, 0, 0] if expect[0] else [math.pi / 2, 0, 0], atol=1e-12)


def test_prop3_closed_form_condition2_and_chain():
    """Closed form, second condition: S = span(e1, e2 + δe5, e3) with δ² = 0.8 > (λ2 − λ3)/(λ3 − λ5) = 2/3:
    on the complement of π_S(e1) = e1 the maximiser is e3, not π_S(e2) ∝ e2 + δe5 (angle π/2); the third
    condition holds on its own (angle 0) but the chain is broken, so its flag is false (reading R28)."""
    X = _diag_data([10, 6, 4, 2, 1, 0.5])
    d = math.sqrt(0.8)
    V = np.array([[1, 0, 0, 0, 0, 0], [0, 1, 0, 0, d, 0], [0, 0, 1, 0, 0, 0]], dtype=np.float64)
    flags, ang = O.check_prop3(X, V, np.eye(6), 3)
    assert flags == [True, False, False]
    np.testing.assert_allclose(ang, [0, math.pi / 2, 0], atol=1e-12)


def test_prop3_condition1_matches_refine():
    """Independent path: condition 1's angle is ∠(first pPCA vector, π_S(e1)) — the refine's Jacobi solve
    lifted to R^d against the projection of the true eigenvector computed here with lstsq."""
    X = _random_data(1500, 8, 41)
    lam, T = O.truth(X)
    rng = np.random.default_rng(42)
    for trial in range(5):
        V = T[:3] + 0.05 * rng.standard_normal((3, 8))
        _, ang = O.check_prop3(X, V, T, 1)
        E, _, _, _ = O.ppca_refine(X, V, 1)
        coef = np.linalg.lstsq(V.T, T[0], rcond=None)[0]
        p = V.T @ coef                                      # π_S(e1)
        p /= np.linalg.norm(p)
        a = math.acos(min(1.0, abs(float(E[0] @ p))))
        assert ang[0] == pytest.approx(a, abs=1e-7)


def test_prop3_degenerate_projection():
    """S L343: π_S(e1) = 0 (S ⊥ e1) raises DegenerateProjection."""
    X = _diag_data([5, 3, 2, 1])
    V = np.array([[0, 1.0, 0, 0], [0, 0, 1.0, 0]])
    with pytest.raises(O.DegenerateProjection):
        O.check_prop3(X, V, np.eye(4), 2)
