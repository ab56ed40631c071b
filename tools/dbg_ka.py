"""Kernel A (refine pass) timing under experiment switches: PPCA_DBG bits (tc_xw.cuh)
1 skip MMA, 2 skip S epilogue, 4 converters skip STS, 8 skip the X_lo MMA, 16 converters store hi only."""
import sys, torch
sys.path.insert(0, '.')
import paper_2109_03709_b200 as P
from inputs import configs as C
ctx = P.ppca_ctx_create(0, torch.cuda.current_stream())
P.ppca_set_pass_impl(ctx, 2)
w = C.C3; s = w.spec
X = torch.empty((s.n, s.d), dtype=torch.float32, device='cuda')
P.ppca_generate(ctx, P.gen_spec(s), X)
Xm = P.matrix(X)
g = torch.Generator(device='cuda').manual_seed(0)
W = torch.randn((w.m, s.d), device='cuda', generator=g)
E = torch.empty((w.k, s.d), device='cuda')
P.ppca_set_timing(ctx, True)
for it in range(2):
    try: P.ppca_refine(ctx, Xm, W, w.m, w.k, E)
    except P.PPCAError: pass
P.ppca_get_pass_time(ctx)
for it in range(3):
    try: P.ppca_refine(ctx, Xm, W, w.m, w.k, E)
    except P.PPCAError: pass
ms, n = P.ppca_get_pass_time(ctx)
print(f"PPCA_DBG={sys.argv[1] if len(sys.argv)>1 else 0}: refine pass (kernel A) {ms/n:.3f} ms  {4096/(ms/n):.0f} GB/s")
