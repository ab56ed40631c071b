"""Seeded synthetic datasets for the five BASELINE.json workloads (host side).

Input generator only (no pPCA arithmetic).  Used by `tests/` and by the oracle
runs; the CUDA library implements the same recipe on the device
(`ppca_generate`, csrc/gen.cu) and `tests/test_gpu_generate.py` compares the two
on sampled rows.  Recipe (BASELINE.json configs[0..4];
PAPER.md §5.1 L365-366 for the planted-spectrum idea):

  planted_qr          x = Q (sqrt(λ) ∘ g),  Q = Q-factor of Γ (d x d iid N(0,1)) with diag(R) > 0
  planted_householder x = max(0, H_1 ... H_r (sqrt(λ) ∘ g)),  H_i = I - 2 u_i u_iᵀ, u_i = γ_i/‖γ_i‖
  image_factor        x = mask ∘ clip((0.13/50)·a·B, 0, 1)  with a (1 x 50 per row) and B (50 x d)
                      iid Exp(1), mask_j = 0 with probability 0.8 (U_j < 0.8)
then column-centred with the fp64 mean over all n rows, and rounded (RNE) to the
storage type (fp32 or bf16).  λ_j is indexed j = 1..d.
"""
from __future__ import annotations

import dataclasses
import functools
import numpy as np

from . import philox as ph


@dataclasses.dataclass(frozen=True)
class GenSpec:
    family: str            # 'planted_qr' | 'planted_householder' | 'image_factor'
    n: int
    d: int
    seed: int
    spectrum: str = "exp"  # 'exp': λ_j = exp(-j/a);  'power': λ_j = j^-a
    a: float = 1.0
    noise: float = 0.0     # added to every λ_j (isotropic noise variance, reading R5)
    relu: bool = False
    house_r: int = 8
    rank: int = 50         # image_factor inner dimension
    dtype: str = "f32"     # storage: 'f32' | 'bf16'

    def lambdas(self) -> np.ndarray:
        j = np.arange(1, self.d + 1, dtype=np.float64)
        if self.spectrum == "exp":
            lam = np.exp(-j / self.a)
        elif self.spectrum == "power":
            lam = j ** (-self.a)
        else:
            raise ValueError(self.spectrum)
        return lam + self.noise


# ----------------------------------------------------------------------------- storage rounding
def f64_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp64 -> bf16 (returned as uint16 bit patterns)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    b = x.view(np.uint64)
    lsb = (b >> np.uint64(45)) & np.uint64(1)
    r = (b + np.uint64((1 << 44) - 1) + lsb) & ~np.uint64((1 << 45) - 1)
    f = r.view(np.float64).astype(np.float32)          # exact: 8 significant bits
    return (f.view(np.uint32) >> np.uint32(16)).astype(np.uint16)


def bf16_bits_to_f64(h: np.ndarray) -> np.ndarray:
    return (np.asarray(h, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)


def store(x: np.ndarray, dtype: str) -> np.ndarray:
    """Stored representation: float32 array for 'f32', uint16 bits for 'bf16'."""
    if dtype == "f32":
        return x.astype(np.float32)
    if dtype == "bf16":
        return f64_to_bf16_bits(x)
    raise ValueError(dtype)


def stored_to_f64(s: np.ndarray, dtype: str) -> np.ndarray:
    return s.astype(np.float64) if dtype == "f32" else bf16_bits_to_f64(s)


# ----------------------------------------------------------------------------- global factors
@functools.lru_cache(maxsize=4)
def planted_q(seed: int, d: int) -> np.ndarray:
    """Haar orthogonal Q: Q-factor of Γ (row-major, stream 1) with positive diag(R)."""
    gam = ph.gaussians(seed, ph.STREAM_GAMMA, 0, d * d).reshape(d, d)
    q, r = np.linalg.qr(gam)
    q = q * np.sign(np.diag(r))[None, :]
    q.setflags(write=False)
    return q


@functools.lru_cache(maxsize=4)
def householder_vectors(seed: int, d: int, r: int) -> np.ndarray:
    u = ph.gaussians(seed, ph.STREAM_HOUSE, 0, r * d).reshape(r, d)
    u = u / np.linalg.norm(u, axis=1, keepdims=True)
    u.setflags(write=False)
    return u


@functools.lru_cache(maxsize=4)
def image_b(seed: int, d: int, rank: int) -> np.ndarray:
    b = ph.exponentials(seed, ph.STREAM_B, 0, rank * d).reshape(rank, d)
    b.setflags(write=False)
    return b


# ----------------------------------------------------------------------------- raw rows
def _runs(rows: np.ndarray):
    """Split sorted-or-not global row indices into maximal contiguous runs (start, len, pos)."""
    rows = np.asarray(rows, dtype=np.int64)
    if rows.size == 0:
        return
    brk = np.nonzero(np.diff(rows) != 1)[0] + 1
    starts = np.concatenate([[0], brk])
    ends = np.concatenate([brk, [rows.size]])
    for s, e in zip(starts, ends):
        yield int(rows[s]), int(e - s), int(s)


def raw_rows(spec: GenSpec, rows) -> np.ndarray:
    """fp64 raw (uncentred) rows for the given global row indices."""
    rows = np.asarray(rows, dtype=np.int64)
    d = spec.d
    out = np.empty((rows.size, d), dtype=np.float64)
    if spec.family in ("planted_qr", "planted_householder"):
        sl = np.sqrt(spec.lambdas())
        for r0, cnt, pos in _runs(rows):
            g = ph.gaussians(spec.seed, ph.STREAM_G, r0 * d, cnt * d).reshape(cnt, d)
            v = g * sl[None, :]
            if spec.family == "planted_qr":
                v = v @ planted_q(spec.seed, d).T
            else:
                u = householder_vectors(spec.seed, d, spec.house_r)
                for i in range(spec.house_r - 1, -1, -1):       # apply H_r first
                    v = v - 2.0 * np.outer(v @ u[i], u[i])
            if spec.relu:
                v = np.maximum(v, 0.0)
            out[pos:pos + cnt] = v
    elif spec.family == "image_factor":
        bm = image_b(spec.seed, d, spec.rank)
        scale = 0.13 / spec.rank
        for r0, cnt, pos in _runs(rows):
            a = ph.exponentials(spec.seed, ph.STREAM_A, r0 * spec.rank, cnt * spec.rank).reshape(cnt, spec.rank)
            p = np.clip(scale * (a @ bm), 0.0, 1.0)
            keep = ph.uniforms(spec.seed, ph.STREAM_MASK, r0 * d, cnt * d).reshape(cnt, d) >= 0.8
            out[pos:pos + cnt] = np.where(keep, p, 0.0)
    else:
        raise ValueError(spec.family)
    return out


_MEAN_CACHE: dict = {}


def column_mean(spec: GenSpec, chunk: int = 16384) -> np.ndarray:
    """fp64 column mean of the raw data over all n rows (chunked, fixed order)."""
    key = spec
    if key in _MEAN_CACHE:
        return _MEAN_CACHE[key]
    acc = np.zeros(spec.d)
    for r0 in range(0, spec.n, chunk):
        r1 = min(spec.n, r0 + chunk)
        acc += raw_rows(spec, np.arange(r0, r1)).sum(axis=0)
    mu = acc / spec.n
    _MEAN_CACHE[key] = mu
    return mu


def stored_rows(spec: GenSpec, rows) -> np.ndarray:
    """Stored X rows: RNE(raw - mean) in the storage type (float32 / uint16 bf16 bits)."""
    return store(raw_rows(spec, rows) - column_mean(spec)[None, :], spec.dtype)


def dataset(spec: GenSpec) -> np.ndarray:
    """Whole stored X (n x d) — small configs only."""
    return stored_rows(spec, np.arange(spec.n))


def dataset_f64(spec: GenSpec) -> np.ndarray:
    """Whole stored X converted exactly to fp64 (what the oracle computes on)."""
    return stored_to_f64(dataset(spec), spec.dtype)


def init_gaussians(init_seed: int, m: int, d: int) -> np.ndarray:
    """Raw N(0,1) draws for the m initial priming vectors, [m][d] (stream 6, index c*d + j)."""
    return ph.gaussians(init_seed, ph.STREAM_INIT, 0, m * d).reshape(m, d)


# ----------------------------------------------------------------------------- row layouts
def shard_rows(n: int, rank: int, world: int, layout: str = "contiguous", block_rows: int = 0) -> np.ndarray:
    """Global row indices stored by `rank`.

    contiguous:  rows [⌈n/G⌉·g, min(n, ⌈n/G⌉·(g+1)))
    interleaved: every minibatch block s = rows [s·b, min(n,(s+1)·b)) of size p is split in G equal
                 slices; rank g stores [s·b + g·p/G, s·b + (g+1)·p/G).  Requires G | p for every block.
    """
    if layout == "contiguous":
        per = -(-n // world)
        return np.arange(min(n, per * rank), min(n, per * (rank + 1)), dtype=np.int64)
    if layout == "interleaved":
        b = block_rows
        out = []
        for s0 in range(0, n, b):
            p = min(b, n - s0)
            if p % world:
                raise ValueError(f"block of {p} rows not divisible by world={world}")
            q = p // world
            out.append(np.arange(s0 + rank * q, s0 + (rank + 1) * q, dtype=np.int64))
        return np.concatenate(out) if out else np.zeros(0, np.int64)
    raise ValueError(layout)
