"""Profiling driver: generate a config on cuda:0, run `iters` power iterations and one refine through
the C ABI.  Used under ncu (launch list / --set full) and for quick CUDA-event timing of the pass.

    python tools/prof_pass.py [C3|C5|C4] [iters] [impl]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2109_03709_b200 as P  # noqa: E402
from inputs import configs as C  # noqa: E402

if os.environ.get("PPCA_EXP_LIB"):               # experiment build (tools/ ablations only)
    P.load(os.environ["PPCA_EXP_LIB"])
name = sys.argv[1] if len(sys.argv) > 1 else "C3"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
impl = int(sys.argv[3]) if len(sys.argv) > 3 else 2
split = len(sys.argv) > 4 and sys.argv[4] == "split"
w = C.FULL[name]
s = w.spec
ctx = P.ppca_ctx_create(0, torch.cuda.current_stream())
P.ppca_set_pass_impl(ctx, impl)
dt = torch.float32 if s.dtype == "f32" else torch.bfloat16
X = torch.empty((s.n, s.d), dtype=dt, device="cuda")
split = split and s.dtype == "f32"
P.ppca_generate(ctx, P.gen_spec(s, split=split), X)
Xm = P.matrix(X, split=split)
W = torch.empty((w.m, s.d), device="cuda")
P.ppca_prime_power(ctx, Xm, w.m, 1, w.init_seed, W)
E = torch.empty((w.k, s.d), device="cuda")
P.ppca_set_timing(ctx, True)
P.ppca_get_pass_time(ctx)
P.ppca_prime_power(ctx, Xm, w.m, iters, 0, W)
ms_p, n_p = P.ppca_get_pass_time(ctx)
P.ppca_refine(ctx, Xm, W, w.m, w.k, E)          # first call: scratch growth for the refine shapes
P.ppca_get_pass_time(ctx)
for _ in range(3):
    P.ppca_refine(ctx, Xm, W, w.m, w.k, E)
ms_r, n_r = P.ppca_get_pass_time(ctx)
gb = s.n * s.d * (4 if s.dtype == "f32" else 2) / 1e9
print(f"{name}{' split' if split else ''}: power pass {ms_p / max(n_p, 1):.3f} ms ({gb / (ms_p / max(n_p, 1)) * 1e3:.0f} GB/s); "
      f"refine pass {ms_r / max(n_r, 1):.3f} ms ({gb / (ms_r / max(n_r, 1)) * 1e3:.0f} GB/s)")
P.ppca_ctx_destroy(ctx)
