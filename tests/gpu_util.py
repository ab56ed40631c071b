"""Helpers for the GPU parity tests (host inputs → device tensors; parity criteria)."""
import math

import numpy as np

from inputs import generate as G
from oracle import ppca_oracle as O

THRESHOLDS = O.PI_THRESHOLDS


def upload(x_stored: np.ndarray, dtype: str, ld: int | None = None):
    """Stored host X (float32 or uint16 bf16 bits) → CUDA tensor [n][ld] (zero padding columns)."""
    import torch
    n, d = x_stored.shape
    elt = 4 if dtype == "f32" else 2
    if ld is None:
        ld = d if (d * elt) % 16 == 0 else d + (16 // elt - (d % (16 // elt)))
    if dtype == "f32":
        t = torch.zeros((n, ld), dtype=torch.float32)
        t[:, :d] = torch.from_numpy(np.ascontiguousarray(x_stored, dtype=np.float32))
    else:
        t = torch.zeros((n, ld), dtype=torch.int16)
        t[:, :d] = torch.from_numpy(np.ascontiguousarray(x_stored).view(np.int16))
        t = t.view(torch.bfloat16)
    return t.cuda()


def ritz_rel_err(th_gpu, th_ref):
    th_gpu, th_ref = np.asarray(th_gpu), np.asarray(th_ref)
    return np.max(np.abs(th_gpu - th_ref) / np.abs(th_ref))


def gapped(lam, k, tol=1e-2):
    g = O.relative_gaps(np.asarray(lam)[: k + 1])[:k]
    return np.nonzero(g > tol)[0]


def abs_cos(E1, E2):
    E1 = np.asarray(E1, dtype=np.float64)
    E2 = np.asarray(E2, dtype=np.float64)
    return np.abs(np.sum(E1 * E2, axis=1)) / (np.linalg.norm(E1, axis=1) * np.linalg.norm(E2, axis=1))


def lces_all(E, T):
    ang = O.angles(np.asarray(E, dtype=np.float64) / np.linalg.norm(E, axis=1, keepdims=True), T)
    return [O.lces(ang, V) for V in THRESHOLDS], ang


def assert_ppca_parity(E_gpu, th_gpu, E_ref, th_ref, T, rtol, what="", th_all_ref=None):
    """North-star parity bar: Ritz values within rtol; |cos| ≥ 0.9999 where the relative gap of the
    reference Ritz values exceeds 1e-2; identical LCES against the truth T at every threshold."""
    k = len(th_ref)
    err = ritz_rel_err(th_gpu, th_ref)
    assert err <= rtol, f"{what}: Ritz rel err {err:.3e} > {rtol}"
    idx = gapped(th_all_ref if th_all_ref is not None else th_ref, k)
    if idx.size:
        cos = abs_cos(E_gpu[idx], E_ref[idx])
        assert cos.min() >= 0.9999, f"{what}: min |cos| {cos.min():.6f} on gapped vectors {idx.tolist()}"
    l_gpu, a_gpu = lces_all(E_gpu, T[:k])
    l_ref, a_ref = lces_all(E_ref, T[:k])
    assert l_gpu == l_ref, f"{what}: LCES gpu {l_gpu} vs oracle {l_ref}"
    return err
