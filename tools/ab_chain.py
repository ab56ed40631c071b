"""Step-level A/B timing (CUDA events, no ncu): C3 power step with the θ history (the bench's step), the C3
refine with the orthonormal flag, and the C4 EigenGame step.  Run once per build / switch setting, e.g.

    PPCA_EXP_LIB=paper_2109_03709_b200/libppca_exp.so PPCA_PDL=0 python tools/ab_chain.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2109_03709_b200 as P  # noqa: E402
from inputs import configs as C  # noqa: E402

if os.environ.get("PPCA_EXP_LIB"):
    P.load(os.environ["PPCA_EXP_LIB"])
which = sys.argv[1:] or ["C3", "C4"]
tag = os.environ.get("AB_TAG", "")
ctx = P.ppca_ctx_create(0, torch.cuda.current_stream())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    best = []
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best.append(e0.elapsed_time(e1))
    best.sort()
    return best[len(best) // 2]


for cname in [c for c in ("C3", "C5") if c in which]:
    w = C.FULL[cname]
    s = w.spec
    bf = s.dtype == "bf16"
    X = torch.empty((s.n, s.d), dtype=torch.bfloat16 if bf else torch.float32, device="cuda")
    P.ppca_generate(ctx, P.gen_spec(s, split=not bf), X)
    Xm = P.matrix(X, split=not bf)
    W = torch.empty((w.m, s.d), device="cuda")
    E = torch.empty((w.k, s.d), device="cuda")
    P.ppca_prime_power(ctx, Xm, w.m, 2, w.init_seed, W)
    it = 10 if cname == "C3" else 4
    ms = timed(lambda: P.ppca_prime_power(ctx, Xm, w.m, it, 0, W, theta_hist=True), 5) / it
    ms_nh = timed(lambda: P.ppca_prime_power(ctx, Xm, w.m, it, 0, W), 5) / it
    P.ppca_set_timing(ctx, True)
    P.ppca_get_pass_time(ctx)
    P.ppca_get_kernel_time(ctx, 0), P.ppca_get_kernel_time(ctx, 1)
    P.ppca_prime_power(ctx, Xm, w.m, it, 0, W)
    pms, npass = P.ppca_get_pass_time(ctx)
    ka, kan = P.ppca_get_kernel_time(ctx, 0)
    kb, kbn = P.ppca_get_kernel_time(ctx, 1)
    print(f"{tag} {cname}: kernel A {ka / max(kan, 1) * 1e3:.1f} us x{kan}, kernel B {kb / max(kbn, 1) * 1e3:.1f} us x{kbn}")
    P.ppca_set_timing(ctx, False)
    rms = timed(lambda: P.ppca_refine_ex(ctx, Xm, W, w.m, w.k, E, flags=1), 5)
    print(f"{tag} {cname}: step {ms * 1e3:.1f} us (theta hist), {ms_nh * 1e3:.1f} us (no hist), pass {pms / npass * 1e3:.1f} us, "
          f"outside pass {(ms_nh - pms / npass) * 1e3:.1f} us; refine_ex(orthonormal) {rms * 1e3:.1f} us", flush=True)
    del X, Xm
    torch.cuda.empty_cache()

if "C4" in which:
    w = C.FULL["C4"]
    s = w.spec
    X = torch.empty((s.n, s.d), dtype=torch.float32, device="cuda")
    P.ppca_generate(ctx, P.gen_spec(s, split=True), X)
    Xm = P.matrix(X, split=True)
    V = torch.empty((w.m, s.d), device="cuda")
    vel = torch.zeros_like(V)
    st = P.ppca_prime_eigengame(ctx, Xm, w.m, w.batch, w.alpha, w.momentum, 5, w.init_seed, V, vel, 0)
    steps = 50
    holder = [st]

    def run():
        holder[0] = P.ppca_prime_eigengame(ctx, Xm, w.m, w.batch, w.alpha, w.momentum, steps, 0, V, vel, holder[0])

    ms = timed(run, 5) / steps
    print(f"{tag} C4: eigengame step {ms * 1e3:.1f} us", flush=True)
    del X, Xm
    torch.cuda.empty_cache()

if "C2" in which:
    w = C.FULL["C2"]
    s = w.spec
    X = torch.empty((s.n, s.d), dtype=torch.float32, device="cuda")
    P.ppca_generate(ctx, P.gen_spec(s, split=True), X)
    Xm = P.matrix(X, split=True)
    V = torch.empty((w.m, s.d), device="cuda")
    vel = torch.zeros_like(V)
    st = P.ppca_prime_oja(ctx, Xm, w.m, w.batch, w.alpha, w.momentum, 5, w.init_seed, V, vel, 0)
    steps = 200
    holder = [st]

    def run2():
        holder[0] = P.ppca_prime_oja(ctx, Xm, w.m, w.batch, w.alpha, w.momentum, steps, 0, V, vel, holder[0])

    ms = timed(run2, 5) / steps
    print(f"{tag} C2: oja step {ms * 1e3:.2f} us", flush=True)
P.ppca_ctx_destroy(ctx)
