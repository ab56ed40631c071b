import sys, time, torch
sys.path.insert(0, '.')
import paper_2109_03709_b200 as P
from inputs import configs as C
ctx = P.ppca_ctx_create(0, torch.cuda.current_stream())
P.ppca_set_pass_impl(ctx, 2)
w = C.C3; s = w.spec
X = torch.empty((s.n, s.d), dtype=torch.float32, device='cuda')
P.ppca_generate(ctx, P.gen_spec(s), X)
Xm = P.matrix(X)
W = torch.empty((w.m, s.d), device='cuda')
P.ppca_prime_power(ctx, Xm, w.m, 1, w.init_seed, W)
E = torch.empty((w.k, s.d), device='cuda')
P.ppca_set_timing(ctx, True)
for it in range(2): P.ppca_refine(ctx, Xm, W, w.m, w.k, E)
P.ppca_get_pass_time(ctx)
for it in range(3): P.ppca_refine(ctx, Xm, W, w.m, w.k, E)
ms, n = P.ppca_get_pass_time(ctx)
print(f"PPCA_DBG={sys.argv[1] if len(sys.argv)>1 else 0}: refine pass (kernel A) {ms/n:.3f} ms  {4096/(ms/n):.0f} GB/s")
