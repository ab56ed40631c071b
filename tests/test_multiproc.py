"""world_size-2 `gloo` tests of the N>1 host logic (CPU, no GPU):

* the CONTIGUOUS shard map of the binding partitions the rows (ppca.h / DESIGN.md §6);
* the NCCL unique-id bootstrap delivers rank 0's bytes to every rank;
* the only exchange of the method is the sum of per-rank partials (P L260–269: XᵀX = Σ_rows xxᵀ):
  per-rank [Z_g | S_g] all-reduced equals the single-process power pass, and the INTERLEAVED block
  schedule (reading R10) reproduces the global minibatch's Oja gradient for any G.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from inputs import generate as G
from oracle import ppca_oracle as O

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fn_name, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        globals()[fn_name](rank, world)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def _run(fn_name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, WORLD, port, fn_name, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(r[1] == "ok" for r in res), res


# ----------------------------------------------------------------------------- rank bodies
def _body_shards(rank, world):
    import torch
    import torch.distributed as dist
    import paper_2109_03709_b200 as P
    for n in (0, 1, 7, 2000, 100003):
        r0, rows = P.contiguous_shard(n, rank, world)
        np.testing.assert_array_equal(np.arange(r0, r0 + rows), G.shard_rows(n, rank, world, "contiguous"))
        cnt = torch.tensor([rows], dtype=torch.int64)
        dist.all_reduce(cnt)
        assert int(cnt) == n
        got = [None] * world
        dist.all_gather_object(got, (r0, rows))
        assert got[0][0] == 0 and all(got[i][0] + got[i][1] == got[i + 1][0] for i in range(world - 1))


def _body_uid(rank, world):
    import paper_2109_03709_b200 as P
    uid = bytes(range(P.PPCA_UNIQUE_ID_BYTES)) if rank == 0 else None
    got = P.broadcast_unique_id(uid)
    assert got == bytes(range(P.PPCA_UNIQUE_ID_BYTES))


def _partials(Xg, W):
    Y = Xg @ W.T
    return Y.T @ Xg, Y.T @ Y


def _body_power_exchange(rank, world):
    import torch
    import torch.distributed as dist
    rng = np.random.default_rng(3)
    n, d, m = 1001, 40, 6
    X = rng.standard_normal((n, d)) * np.exp(-np.arange(d) / 8)
    W = O.gram_schmidt(rng.standard_normal((m, d)), drop=False)
    rows = G.shard_rows(n, rank, world, "contiguous")
    Zg, Sg = _partials(X[rows], W)
    buf = torch.from_numpy(np.concatenate([Zg.ravel(), Sg.ravel()]))
    dist.all_reduce(buf)                                  # the method's only collective
    Z = buf[: m * d].numpy().reshape(m, d)
    S = buf[m * d:].numpy().reshape(m, m)
    W_ref, S_ref = O.power_step(X, W)
    np.testing.assert_allclose(S, S_ref, rtol=1e-12)
    np.testing.assert_allclose(O.gram_schmidt(Z, drop=False), W_ref, atol=1e-12)


def _body_oja_interleaved(rank, world):
    import torch
    import torch.distributed as dist
    rng = np.random.default_rng(4)
    n, d, m, b = 1000, 24, 4, 128                         # last block 1000 − 7·128 = 104 rows
    X = rng.standard_normal((n, d))
    W = rng.standard_normal((m, d))
    mine = G.shard_rows(n, rank, world, "interleaved", b)
    blocks = O.minibatch_blocks(n, b)
    for s in (0, 3, len(blocks) - 1):
        r0, r1 = blocks[s]
        local = mine[(mine >= r0) & (mine < r1)]
        assert local.size == (r1 - r0) // world
        Y = X[local] @ W.T
        buf = torch.from_numpy(np.concatenate([(Y.T @ X[local]).ravel(), (Y.T @ Y).ravel()]))
        dist.all_reduce(buf)
        XtY = buf[: m * d].numpy().reshape(m, d)
        YtY = buf[m * d:].numpy().reshape(m, m)
        G_dist = XtY - np.tril(YtY) @ W                   # Σ_{l ≤ m} (Sanger, P L70–72)
        W_ref, v_ref = O.oja_step(X[r0:r1], W, np.zeros_like(W), 1e-3, 0.0)
        np.testing.assert_allclose(W + 1e-3 * G_dist, W_ref, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("body", ["_body_shards", "_body_uid", "_body_power_exchange", "_body_oja_interleaved"])
def test_gloo_world2(body):
    _run(body)
