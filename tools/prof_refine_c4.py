"""Time the pieces of the C4 time-to-LCES loop: minibatch EigenGame steps and full refines (CUDA events)."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2109_03709_b200 as P  # noqa: E402
from inputs import configs as C  # noqa: E402
w = C.FULL[sys.argv[1] if len(sys.argv) > 1 else "C4"]
s = w.spec
ctx = P.ppca_ctx_create(0, torch.cuda.current_stream())
X = torch.empty((s.n, s.d), dtype=torch.float32, device="cuda")
P.ppca_generate(ctx, P.gen_spec(s, split=True), X)
Xm = P.matrix(X, split=True)
V = torch.empty((w.m, s.d), device="cuda"); vel = torch.zeros_like(V)
E = torch.empty((w.k, s.d), device="cuda")
fn = P.ppca_prime_oja if w.priming == "oja" else P.ppca_prime_eigengame
step = fn(ctx, Xm, w.m, w.batch, w.alpha, w.momentum, 0, w.init_seed, V, vel, 0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for cp in [16, 32, 64, 128, 256]:
    e0.record(); step = fn(ctx, Xm, w.m, w.batch, w.alpha, w.momentum, cp - step, 0, V, vel, step); e1.record()
    torch.cuda.synchronize(); ts = e0.elapsed_time(e1)
    t0 = time.time(); e0.record(); P.ppca_refine(ctx, Xm, V, w.m, w.k, E); e1.record()
    torch.cuda.synchronize(); tr = e0.elapsed_time(e1)
    print(f"checkpoint {cp}: steps {ts:.2f} ms, refine {tr:.2f} ms (host {1e3 * (time.time() - t0):.1f} ms)")
