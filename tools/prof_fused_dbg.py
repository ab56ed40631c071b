"""Fused-pass experiments: time one power pass (kernel events) under PPCA_DBG switches, ignoring the
numerical failure a disabled stage causes downstream."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2109_03709_b200 as P
from inputs import configs as C
w = C.C3; s = w.spec
ctx = P.ppca_ctx_create(0, torch.cuda.current_stream())
P.ppca_set_pass_impl(ctx, 2)
X = torch.empty((s.n, s.d), dtype=torch.float32, device="cuda")
P.ppca_generate(ctx, P.gen_spec(s, split=True), X)
Xm = P.matrix(X, split=True)
g = torch.Generator(device="cuda").manual_seed(0)
W = torch.linalg.qr(torch.randn((s.d, w.m), device="cuda", generator=g))[0].T.contiguous()
P.ppca_set_timing(ctx, True)
tot, n = 0.0, 0
for it in range(6):
    W2 = W.clone()
    try:
        P.ppca_prime_power(ctx, Xm, w.m, 1, 0, W2)
    except P.PPCAError:
        pass
    ms, k = P.ppca_get_kernel_time(ctx, 0)
    if it >= 2:
        tot += ms; n += k
print(f"PPCA_DBG={os.environ.get('PPCA_DBG', '0')}: fused kernel {tot / max(n, 1):.3f} ms ({4.096 / (tot / max(n, 1)):.0f} GB/s)")
