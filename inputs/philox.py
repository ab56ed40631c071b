"""Counter-based random numbers for the seeded synthetic inputs (host side).

This module is the *input generator* shared by the tests and the oracle side.
It holds none of the pPCA arithmetic: it only turns (seed, stream, index)
into uint32 words, uniforms, Gaussians and Exp(1) draws.  The CUDA library
(`paper_2109_03709_b200/csrc/gen.cu`) implements the same generator
independently on the device; `tests/test_gpu_generate.py` checks that both
produce the same values element by element.

Philox4x32-10 (Salmon et al., SC'11 "Parallel random numbers: as easy as
1, 2, 3"): a 4x32-bit counter, a 2x32-bit key, 10 rounds, key bumped by the
Weyl constants between rounds.  The same function is the CUDA toolkit's
`curand_Philox4x32_10(uint4 ctr, uint2 key)`.

Counter convention used by every input of this repo:
    ctr = (call_index_lo32, call_index_hi32, stream, 0),  key = (seed_lo32, seed_hi32)
one call yields 4 words; element e of a stream uses word e % 4 of call e // 4.
"""
from __future__ import annotations

import numpy as np

PHILOX_M0 = np.uint64(0xD2511F53)
PHILOX_M1 = np.uint64(0xCD9E8D57)
PHILOX_W0 = np.uint32(0x9E3779B9)
PHILOX_W1 = np.uint32(0xBB67AE85)
_MASK32 = np.uint64(0xFFFFFFFF)

# stream ids
STREAM_G = 0          # data Gaussians g (planted families)
STREAM_GAMMA = 1      # Gaussian seed matrix Γ whose QR factor is Q
STREAM_HOUSE = 2      # Householder vectors u_i
STREAM_A = 3          # image factor A (n x 50), Exp(1)
STREAM_B = 4          # image factor B (50 x d), Exp(1)
STREAM_MASK = 5       # image mask uniforms
STREAM_INIT = 6       # priming initial vectors


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Vectorised Philox4x32-10.  All inputs uint32 arrays (broadcastable)."""
    c0 = np.asarray(c0, dtype=np.uint32).astype(np.uint64)
    c1 = np.asarray(c1, dtype=np.uint32).astype(np.uint64)
    c2 = np.asarray(c2, dtype=np.uint32).astype(np.uint64)
    c3 = np.asarray(c3, dtype=np.uint32).astype(np.uint64)
    k0 = np.uint32(k0)
    k1 = np.uint32(k1)
    c0, c1, c2, c3 = np.broadcast_arrays(c0, c1, c2, c3)
    for r in range(10):
        p0 = PHILOX_M0 * c0            # exact: both < 2^32
        p1 = PHILOX_M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & _MASK32
        hi1, lo1 = p1 >> np.uint64(32), p1 & _MASK32
        n0 = hi1 ^ c1 ^ np.uint64(k0)
        n1 = lo1
        n2 = hi0 ^ c3 ^ np.uint64(k1)
        n3 = lo0
        c0, c1, c2, c3 = n0, n1, n2, n3
        if r != 9:
            k0 = np.uint32((int(k0) + int(PHILOX_W0)) & 0xFFFFFFFF)
            k1 = np.uint32((int(k1) + int(PHILOX_W1)) & 0xFFFFFFFF)
    return (c0.astype(np.uint32), c1.astype(np.uint32),
            c2.astype(np.uint32), c3.astype(np.uint32))


def words(seed: int, stream: int, first: int, count: int) -> np.ndarray:
    """uint32 words w[e] for e in [first, first+count) of (seed, stream)."""
    if count <= 0:
        return np.zeros(0, dtype=np.uint32)
    c_lo, c_hi = first // 4, (first + count - 1) // 4
    calls = np.arange(c_lo, c_hi + 1, dtype=np.uint64)
    r = philox4x32_10(calls & _MASK32, calls >> np.uint64(32),
                      np.uint32(stream), np.uint32(0),
                      np.uint32(seed & 0xFFFFFFFF), np.uint32((seed >> 32) & 0xFFFFFFFF))
    w = np.stack(r, axis=1).reshape(-1)
    off = first - 4 * c_lo
    return w[off:off + count]


def uniforms(seed: int, stream: int, first: int, count: int) -> np.ndarray:
    """U = (w + 0.5) * 2^-32 in fp64, strictly inside (0, 1)."""
    return (words(seed, stream, first, count).astype(np.float64) + 0.5) * 2.0 ** -32


def uniforms_at(seed: int, stream: int, idx) -> np.ndarray:
    """U at arbitrary element indices idx (uint64-compatible array) of (seed, stream)."""
    idx = np.asarray(idx, dtype=np.uint64).reshape(-1)
    if idx.size == 0:
        return np.zeros(0)
    calls = idx >> np.uint64(2)
    r = philox4x32_10(calls & _MASK32, calls >> np.uint64(32), np.uint32(stream), np.uint32(0),
                      np.uint32(seed & 0xFFFFFFFF), np.uint32((seed >> 32) & 0xFFFFFFFF))
    w = np.stack(r, axis=1)[np.arange(idx.size), (idx & np.uint64(3)).astype(np.int64)]
    return (w.astype(np.float64) + 0.5) * 2.0 ** -32


def gaussians(seed: int, stream: int, first: int, count: int) -> np.ndarray:
    """Box-Muller on word pairs (2j, 2j+1): z_{2j} = r cos(2πu_{2j+1}), z_{2j+1} = r sin(2πu_{2j+1}),
    r = sqrt(-2 ln u_{2j}).  Element e depends only on pair e // 2."""
    if count <= 0:
        return np.zeros(0)
    p0, p1 = first // 2, (first + count - 1) // 2
    u = uniforms(seed, stream, 2 * p0, 2 * (p1 - p0 + 1)).reshape(-1, 2)
    rad = np.sqrt(-2.0 * np.log(u[:, 0]))
    ang = 2.0 * np.pi * u[:, 1]
    z = np.stack([rad * np.cos(ang), rad * np.sin(ang)], axis=1).reshape(-1)
    off = first - 2 * p0
    return z[off:off + count]


def exponentials(seed: int, stream: int, first: int, count: int) -> np.ndarray:
    """Exp(1) = -ln U."""
    return -np.log(uniforms(seed, stream, first, count))
