"""The oracle on the reduced BASELINE workloads: properties the paper fixes (no GPU)."""
import numpy as np

from inputs import configs as C
from inputs import generate as G
from oracle import ppca_oracle as O


def test_c1_power_priming_then_ppca_recovers_top_k():
    w = C.C1
    X = G.dataset_f64(w.spec)
    lam, T = O.truth(X)
    W, S_hist = O.prime_power(X, G.init_gaussians(w.init_seed, w.m, w.spec.d), w.iters)
    np.testing.assert_allclose(W @ W.T, np.eye(w.m), atol=1e-12)
    E, th, th_all, dim = O.ppca_refine(X, W, w.k)
    assert dim == w.m
    ang = O.angles(E, T[: w.k])
    assert O.lces(ang, np.pi / 1024) == w.k
    # interlacing of the Ritz values with the true spectrum (Cauchy)
    d, m = w.spec.d, w.m
    for i in range(m):
        assert lam[i + d - m] * (1 - 1e-12) <= th_all[i] <= lam[i] * (1 + 1e-12)
    # S_t is the pPCA Gram of the iterate: Ritz values of the last S equal the refine of W_{T-1}
    assert len(S_hist) == w.iters
    # pPCA helps: raw power columns are further from the truth than the Ritz vectors
    raw = O.angles(W[: w.k], T[: w.k])
    assert ang.sum() <= raw.sum()


def test_c3s_ppca_beats_raw_power_columns():
    w = C.SMALL["C3s"]
    X = G.dataset_f64(w.spec)
    lam, T = O.truth(X)
    W, _ = O.prime_power(X, G.init_gaussians(w.init_seed, w.m, w.spec.d), w.iters)
    E, th, _, _ = O.ppca_refine(X, W, w.k)
    a_ppca, a_raw = O.angles(E, T[: w.k]), O.angles(W[: w.k], T[: w.k])
    for V in O.PI_THRESHOLDS:
        assert O.lces(a_ppca, V) >= O.lces(a_raw, V)
    assert O.lces(a_ppca, np.pi / 8) == w.k


def test_c2s_oja_sum_with_nesterov_makes_progress():
    w = C.SMALL["C2s"]
    X = G.dataset_f64(w.spec)
    lam, T = O.truth(X)
    W0 = G.init_gaussians(w.init_seed, w.m, w.spec.d)
    W, vel = O.prime_oja(X, W0, w.batch, w.alpha, w.momentum, 150)
    E, th, _, _ = O.ppca_refine(X, W, w.k)
    a_ppca = O.angles(E, T[: w.k])
    a_init = O.angles(O.normalize_rows(W0)[: w.k], T[: w.k])
    assert O.lces(a_ppca, np.pi / 8) >= 1            # the well-gapped top direction is found
    assert a_ppca[0] < 0.1 * a_init[0]


def test_c4s_eigengame_unit_norm_and_progress():
    w = C.SMALL["C4s"]
    X = G.dataset_f64(w.spec)
    lam, T = O.truth(X)
    V, vel = O.prime_eigengame(X, G.init_gaussians(w.init_seed, w.m, w.spec.d), w.batch, w.alpha,
                               w.momentum, 20)
    np.testing.assert_allclose(np.linalg.norm(V, axis=1), 1, atol=1e-12)
    E, th, _, _ = O.ppca_refine(X, V, w.k)
    assert O.angles(E, T[: w.k])[0] < np.pi / 8
