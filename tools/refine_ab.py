"""C3 refine (orthonormal flag, as in bench.py's time-to-LCES) after t power iterations: CUDA-event time of the
whole refine and of the Ritz solve's share.  Run with the experiment build to compare Ritz solvers, e.g.

    PPCA_EXP_LIB=paper_2109_03709_b200/libppca_exp.so PPCA_RITZ_JACOBI=1 python tools/refine_ab.py 4 10
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2109_03709_b200 as P  # noqa: E402
from inputs import configs as C  # noqa: E402

if os.environ.get("PPCA_EXP_LIB"):
    P.load(os.environ["PPCA_EXP_LIB"])
its = [int(a) for a in sys.argv[1:]] or [4, 10]
w = C.FULL["C3"]
s = w.spec
ctx = P.ppca_ctx_create(0, torch.cuda.current_stream())
X = torch.empty((s.n, s.d), dtype=torch.float32, device="cuda")
P.ppca_generate(ctx, P.gen_spec(s, split=True), X)
Xm = P.matrix(X, split=True)
W = torch.empty((w.m, s.d), device="cuda")
E = torch.empty((w.k, s.d), device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
tag = os.environ.get("AB_TAG", "jacobi=" + os.environ.get("PPCA_RITZ_JACOBI", "0"))
for t in its:
    P.ppca_prime_power(ctx, Xm, w.m, t, w.init_seed, W)
    th, _ = P.ppca_refine_ex(ctx, Xm, W, w.m, w.k, E, flags=1)
    torch.cuda.synchronize()
    ts = []
    for _ in range(7):
        e0.record()
        th, _ = P.ppca_refine_ex(ctx, Xm, W, w.m, w.k, E, flags=1)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(f"{tag} t={t}: refine_ex {ts[3] * 1e3:.1f} us (min {ts[0] * 1e3:.1f}); theta[:3] {np.asarray(th)[:3]}", flush=True)
P.ppca_ctx_destroy(ctx)
