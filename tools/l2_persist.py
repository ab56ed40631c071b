"""Experiment: does an L2 set-aside for persisting (evict_last) lines help the C3 pair kernel's X_hi re-reads?
Times the C3 power step (θ history, as bench.py) with cudaLimitPersistingL2CacheSize = 0 and a few set-aside
sizes (CUDA events, no ncu).

    python tools/l2_persist.py [MB ...]
"""
import os
import sys

import torch
from cuda.bindings import runtime as rt

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2109_03709_b200 as P  # noqa: E402
from inputs import configs as C  # noqa: E402

sizes = [int(a) for a in sys.argv[1:]] or [0, 16, 32, 64, 0, 96]
torch.cuda.init()
err, mx = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrMaxPersistingL2CacheSize, 0)
print("max persisting L2 bytes", mx, flush=True)
ctx = P.ppca_ctx_create(0, torch.cuda.current_stream())
w = C.FULL["C3"]
s = w.spec
X = torch.empty((s.n, s.d), dtype=torch.float32, device="cuda")
P.ppca_generate(ctx, P.gen_spec(s, split=True), X)
Xm = P.matrix(X, split=True)
W = torch.empty((w.m, s.d), device="cuda")
P.ppca_prime_power(ctx, Xm, w.m, 2, w.init_seed, W)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
it = 10
for mb in sizes:
    torch.cuda.synchronize()
    b = min(mx, mb << 20)
    print("set", b, rt.cudaDeviceSetLimit(rt.cudaLimit.cudaLimitPersistingL2CacheSize, b), flush=True)
    P.ppca_prime_power(ctx, Xm, w.m, it, 0, W, theta_hist=True)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0.record()
        P.ppca_prime_power(ctx, Xm, w.m, it, 0, W, theta_hist=True)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / it)
    ts.sort()
    print(f"persisting set-aside {mb:4d} MB: step {ts[2] * 1e3:.1f} us (min {ts[0] * 1e3:.1f})", flush=True)
P.ppca_ctx_destroy(ctx)
