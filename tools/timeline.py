"""Live kernel timeline (CUPTI activity records through torch.profiler — no replay, no serialisation) of the
bench's C3 power step: prints every kernel of a few steady-state iterations with its stream, start offset,
duration and the gap before it on its stream.

    python tools/timeline.py [C3|C5] [iters] [hist 0|1]
"""
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2109_03709_b200 as P  # noqa: E402
from inputs import configs as C  # noqa: E402

if os.environ.get("PPCA_EXP_LIB"):
    P.load(os.environ["PPCA_EXP_LIB"])
name = sys.argv[1] if len(sys.argv) > 1 else "C3"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 6
hist = (sys.argv[3] != "0") if len(sys.argv) > 3 else True
w = C.FULL[name]
s = w.spec
bf = s.dtype == "bf16"
ctx = P.ppca_ctx_create(0, torch.cuda.current_stream())
X = torch.empty((s.n, s.d), dtype=torch.bfloat16 if bf else torch.float32, device="cuda")
P.ppca_generate(ctx, P.gen_spec(s, split=not bf), X)
Xm = P.matrix(X, split=not bf)
W = torch.empty((w.m, s.d), device="cuda")
if name in ("C2", "C4"):                         # minibatch priming steps (Oja / EigenGame)
    vel = torch.zeros_like(W)
    fn = P.ppca_prime_oja if name == "C2" else P.ppca_prime_eigengame
    st = fn(ctx, Xm, w.m, w.batch, w.alpha, w.momentum, 5, w.init_seed, W, vel, 0)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn(ctx, Xm, w.m, w.batch, w.alpha, w.momentum, iters, 0, W, vel, st)
        torch.cuda.synchronize()
elif len(sys.argv) > 4 and sys.argv[4] == "refine":    # python tools/timeline.py C3 4 0 refine: one refine after `iters` steps
    E = torch.empty((w.k, s.d), device="cuda")
    P.ppca_prime_power(ctx, Xm, w.m, iters, w.init_seed, W)
    P.ppca_refine_ex(ctx, Xm, W, w.m, w.k, E, flags=1)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        P.ppca_refine_ex(ctx, Xm, W, w.m, w.k, E, flags=1)
        torch.cuda.synchronize()
else:
    P.ppca_prime_power(ctx, Xm, w.m, 2, w.init_seed, W, theta_hist=hist)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        P.ppca_prime_power(ctx, Xm, w.m, iters, 0, W, theta_hist=hist)
        torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
rows = []
for e in evs:
    rows.append((e.time_range.start, e.time_range.end, getattr(e, "device_resource_id", 0) or 0, e.name))
rows.sort()
t0 = rows[0][0]
last_end = {}
pair_starts = [r[0] for r in rows if "pair" in r[3] or "xw_tma" in r[3] or "xwz" in r[3]]
print(f"{name}: {len(rows)} kernels, {iters} iterations (hist={hist}); pass-kernel period(us):",
      [round(b - a, 1) for a, b in zip(pair_starts, pair_starts[1:])])
for st, en, sid, nm in rows:
    gap = st - last_end.get(sid, st)
    last_end[sid] = en
    print(f"{st - t0:10.1f} {en - st:8.1f} gap {gap:7.1f} s{sid:<3} {nm[:90]}")
P.ppca_ctx_destroy(ctx)
