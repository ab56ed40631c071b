"""Experiment build: EigenGame priming (C4s and C4) gives bitwise the same V with and without the operand split
fused into the update kernel (PPCA_EG_PREP=0/1 in two processes; prints a hash of V)."""
import hashlib
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2109_03709_b200 as P  # noqa: E402
from inputs import configs as C  # noqa: E402

P.load(os.environ["PPCA_EXP_LIB"])
ctx = P.ppca_ctx_create(0, torch.cuda.current_stream())
for w in (C.SMALL["C4s"], C.FULL["C4"]):
    s = w.spec
    X = torch.empty((s.n, s.d), dtype=torch.float32, device="cuda")
    P.ppca_generate(ctx, P.gen_spec(s, split=True), X)
    Xm = P.matrix(X, split=True)
    V = torch.empty((w.m, s.d), device="cuda")
    vel = torch.zeros_like(V)
    P.ppca_prime_eigengame(ctx, Xm, w.m, w.batch, w.alpha, w.momentum, 12, w.init_seed, V, vel, 0)
    torch.cuda.synchronize()
    print(f"EG_PREP={os.environ.get('PPCA_EG_PREP')} {w.name}: V sha1 {hashlib.sha1(V.cpu().numpy().tobytes()).hexdigest()}",
          flush=True)
    del X, Xm
    torch.cuda.empty_cache()
P.ppca_ctx_destroy(ctx)
