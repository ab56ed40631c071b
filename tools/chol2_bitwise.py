"""Experiment build: the power loop's W after 6 C3s/C3 iterations is bitwise the same with the one-step and the
two-step Cholesky sweep (PPCA_CHOL2=0/1 in two processes; prints a hash of W)."""
import hashlib
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2109_03709_b200 as P  # noqa: E402
from inputs import configs as C  # noqa: E402

P.load(os.environ["PPCA_EXP_LIB"])
ctx = P.ppca_ctx_create(0, torch.cuda.current_stream())
for w in (C.C1, C.FULL["C3"]):
    s = w.spec
    X = torch.empty((s.n, s.d), dtype=torch.float32, device="cuda")
    split = s.n > 100000
    P.ppca_generate(ctx, P.gen_spec(s, split=split), X)
    Xm = P.matrix(X, split=split)
    W = torch.empty((w.m, s.d), device="cuda")
    P.ppca_prime_power(ctx, Xm, w.m, 6, w.init_seed, W)
    torch.cuda.synchronize()
    print(f"CHOL2={os.environ.get('PPCA_CHOL2')} n={s.n}: W sha1 {hashlib.sha1(W.cpu().numpy().tobytes()).hexdigest()}", flush=True)
    del X, Xm
P.ppca_ctx_destroy(ctx)
