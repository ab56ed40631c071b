import ctypes, sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2109_03709_b200 as P
from inputs import configs as C
lib = P.load()
lib.ppca_debug_wait_counters.argtypes = [ctypes.c_void_p]
ctx = P.ppca_ctx_create(0, torch.cuda.current_stream())
P.ppca_set_pass_impl(ctx, 2)
w = C.C3; s = w.spec
X = torch.empty((s.n, s.d), dtype=torch.float32, device='cuda')
P.ppca_generate(ctx, P.gen_spec(s), X)
Xm = P.matrix(X)
W = torch.empty((w.m, s.d), device='cuda')
P.ppca_prime_power(ctx, Xm, w.m, 1, w.init_seed, W)
buf = (ctypes.c_ulonglong * 16)()
lib.ppca_debug_wait_counters(buf)
E = torch.empty((w.k, s.d), device='cuda')
for it in range(3):
    P.ppca_refine(ctx, Xm, W, w.m, w.k, E)       # kernel A only (refine mode)
lib.ppca_debug_wait_counters(buf)
names = ['prod wempty', 'prodX empty', 'mma tempty', 'mma wfull', 'mma full', 'conv empty', 'epi tfull']
tot = buf[15]
print('kernel cycles (sum over CTAs, thread 0):', tot)
for i, nm in enumerate(names):
    print(f'{nm:12s} {buf[i]:16d}  per-CTA-thread fraction of kernel time: {buf[i] / max(tot,1):.3f}')
