"""Kernel A (refine pass) timing under experiment switches: PPCA_DBG bits (tc_xw.cuh)
1 skip MMA, 2 skip S epilogue, 4 converters skip STS, 8 skip the X_lo MMA, 16 converters store hi only."""
import sys, torch
sys.path.insert(0, '.')
import paper_2109_03709_b200 as P
from inputs import configs as C
ctx = P.ppca_ctx_create(0, torch.cuda.current_stream())
P.ppca_set_pass_impl(ctx, 2)
w = C.C3; s = w.spec
split = len(sys.argv) > 2 and sys.argv[2] == 'split'
X = torch.empty((s.n, s.d), dtype=torch.float32, device='cuda')
P.ppca_generate(ctx, P.gen_spec(s, split=split), X)
Xm = P.matrix(X, split=split)
g = torch.Generator(device='cuda').manual_seed(0)
W = torch.randn((w.m, s.d), device='cuda', generator=g)
E = torch.empty((w.k, s.d), device='cuda')
P.ppca_set_timing(ctx, True)
# captured variance = the refine-mode pass (kernel A) without the Ritz solve (no error on garbage S)
for it in range(2):
    P.ppca_captured_variance(ctx, Xm, W, w.m)
P.ppca_get_pass_time(ctx)
for it in range(3):
    P.ppca_captured_variance(ctx, Xm, W, w.m)
ms, n = P.ppca_get_pass_time(ctx)
print(f"PPCA_DBG={sys.argv[1] if len(sys.argv)>1 else 0} split={split}: refine pass (kernel A) {ms/n:.3f} ms  {4096/(ms/n):.0f} GB/s")
