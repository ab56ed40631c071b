"""The seeded input generator (inputs/) — no GPU."""
import os

import numpy as np
import pytest

from inputs import philox as ph
from inputs import generate as G
from inputs import configs as C
from oracle import ppca_oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_philox_known_answers():
    rows = []
    with open(os.path.join(GOLD, "philox4x32_10_kat.txt")) as f:
        for line in f:
            if line.strip() and not line.startswith("#"):
                rows.append([int(x, 16) for x in line.split()])
    for r in rows:
        out = ph.philox4x32_10(*[np.uint32(x) for x in r[:4]], r[4], r[5])
        assert [int(o) for o in out] == r[6:]


def test_words_indexing_is_offset_invariant():
    w = ph.words(123, 0, 0, 103)
    for first in (0, 1, 5, 50):
        np.testing.assert_array_equal(ph.words(123, 0, first, 30), w[first:first + 30])
    z = ph.gaussians(7, 0, 0, 41)
    np.testing.assert_array_equal(ph.gaussians(7, 0, 3, 11), z[3:14])
    assert not np.array_equal(ph.words(123, 1, 0, 8), w[:8])          # streams differ


def test_gaussian_and_exponential_moments():
    z = ph.gaussians(99, 0, 0, 400_000)
    assert abs(z.mean()) < 5 / np.sqrt(z.size)
    assert abs(z.var() - 1) < 0.01
    assert abs(np.mean(z ** 4) - 3) < 0.05
    e = ph.exponentials(99, 3, 0, 400_000)
    assert abs(e.mean() - 1) < 0.01 and abs(e.var() - 1) < 0.02
    u = ph.uniforms(99, 5, 0, 100_000)
    assert 0 < u.min() and u.max() < 1


def test_bf16_rounding_rne():
    # exact bf16 values round-trip; halfway cases go to even
    vals = np.array([1.0, -2.5, 3.140625, 1e-3, 65504.0])
    bits = G.f64_to_bf16_bits(vals)
    back = G.bf16_bits_to_f64(bits)
    assert np.all(np.abs(back - vals) <= np.abs(vals) * 2 ** -8)
    one = 1.0
    half_ulp = 2 ** -8                                   # bf16 ulp at 1 is 2^-7
    assert G.bf16_bits_to_f64(G.f64_to_bf16_bits(np.array([one + half_ulp])))[0] == 1.0   # tie → even
    assert G.bf16_bits_to_f64(G.f64_to_bf16_bits(np.array([one + 3 * half_ulp])))[0] == 1.0 + 2 ** -6
    assert G.bf16_bits_to_f64(G.f64_to_bf16_bits(np.array([one + half_ulp * 1.0001])))[0] == 1.0 + 2 ** -7
    rng = np.random.default_rng(0)
    x = rng.standard_normal(10000)
    b = G.bf16_bits_to_f64(G.f64_to_bf16_bits(x))
    # nearest: no other bf16 value is closer
    up = G.bf16_bits_to_f64(G.f64_to_bf16_bits(x).astype(np.uint16) + 1)
    dn = G.bf16_bits_to_f64(G.f64_to_bf16_bits(x).astype(np.uint16) - 1)
    assert np.all(np.abs(b - x) <= np.abs(up - x)) and np.all(np.abs(b - x) <= np.abs(dn - x))


def test_planted_q_orthogonal_and_spectrum_recovery():
    spec = C.C1.spec
    Q = G.planted_q(spec.seed, spec.d)
    np.testing.assert_allclose(Q.T @ Q, np.eye(spec.d), atol=1e-12)
    X = G.dataset_f64(spec)
    assert X.shape == (2000, 64)
    np.testing.assert_allclose(X.mean(axis=0), 0, atol=1e-6)
    lam, T = O.truth(X)
    planted = spec.lambdas()
    # T12: eig(XᵀX)/n ≈ λ_j within sampling error (n=2000 ⇒ a few % on the top ones)
    np.testing.assert_allclose(lam[:4] / spec.n, planted[:4], rtol=0.1)
    # and the top eigenvectors are close to the planted columns of Q
    for j in range(3):
        assert abs(T[j] @ Q[:, j]) > 0.95


def test_householder_and_image_factor_stats():
    spec = C.SMALL["C5s"].spec
    U = G.householder_vectors(spec.seed, spec.d, spec.house_r)
    np.testing.assert_allclose(np.linalg.norm(U, axis=1), 1, atol=1e-14)
    raw = G.raw_rows(spec, np.arange(64))
    assert raw.min() == 0.0 and np.mean(raw == 0) > 0.3            # ReLU
    st = G.stored_rows(spec, np.arange(5))
    assert st.dtype == np.uint16
    spec2 = C.C2.spec
    raw2 = G.raw_rows(spec2, np.arange(3000))
    assert 0.75 < np.mean(raw2 == 0) < 0.85                         # 80 % mask
    nz = raw2[raw2 > 0]
    assert 0.11 < nz.mean() < 0.15 and nz.max() <= 1.0             # scaled to mean 0.13


def test_rows_are_row_independent():
    spec = C.SMALL["C3s"].spec
    a = G.raw_rows(spec, np.arange(10, 20))
    b = G.raw_rows(spec, np.array([15, 11, 19]))
    np.testing.assert_allclose(b, a[[5, 1, 9]], rtol=0, atol=1e-14)   # up to fp64 sum order


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_shard_rows_partition(world):
    for n, layout, b in [(20011, "contiguous", 0), (12096, "interleaved", 256), (41216, "interleaved", 4096)]:
        parts = [G.shard_rows(n, g, world, layout, b) for g in range(world)]
        allr = np.sort(np.concatenate(parts))
        np.testing.assert_array_equal(allr, np.arange(n))
        if layout == "interleaved":
            # every global minibatch block is split evenly, in order, across ranks
            for s0 in range(0, n, b):
                p = min(b, n - s0)
                for g in range(world):
                    blk = parts[g][(parts[g] >= s0) & (parts[g] < s0 + p)]
                    assert blk.size == p // world
