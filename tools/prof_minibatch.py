"""Minibatch priming step timing (C2 generalized Oja, C4 EigenGame) through the C ABI on cuda:0.

    python tools/prof_minibatch.py [C2|C4] [steps] [split]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2109_03709_b200 as P  # noqa: E402
from inputs import configs as C  # noqa: E402

if os.environ.get("PPCA_EXP_LIB"):               # experiment build (tools/ ablations only)
    P.load(os.environ["PPCA_EXP_LIB"])
name = sys.argv[1] if len(sys.argv) > 1 else "C4"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
split = len(sys.argv) > 3 and sys.argv[3] == "split"
w = C.FULL[name]
s = w.spec
ctx = P.ppca_ctx_create(0, torch.cuda.current_stream())
X = torch.empty((s.n, s.d), dtype=torch.float32, device="cuda")
P.ppca_generate(ctx, P.gen_spec(s, split=split), X)
Xm = P.matrix(X, split=split)
W = torch.empty((w.m, s.d), device="cuda")
V = torch.zeros_like(W)
fn = P.ppca_prime_oja if w.priming == "oja" else P.ppca_prime_eigengame
fn(ctx, Xm, w.m, w.batch, w.alpha, w.momentum, 5, w.init_seed, W, V, 0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
l0 = P.ppca_launch_count(ctx)
e0.record()
fn(ctx, Xm, w.m, w.batch, w.alpha, w.momentum, steps, 0, W, V, 5)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
mb = w.batch * s.d * 4 / 1e6
print(f"{name}{' split' if split else ''}: {ms * 1e3:.1f} us/step  ({mb:.1f} MB of X per step -> {mb / ms:.1f} GB/s), "
      f"{(P.ppca_launch_count(ctx) - l0) / steps:.1f} launches/step")
