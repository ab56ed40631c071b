"""Small runs of every hot-path kernel family for compute-sanitizer (memcheck / racecheck / synccheck):
the d-sliced pair power pass (DSMEM bulk-copy exchange), the row-group fused pass (cross-CTA flag protocol),
the two-kernel pass, the K-split refine, the
persistent cooperative Oja kernel, the EigenGame window pass + cooperative update, the m×m chain.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import dataclasses
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2109_03709_b200 as P  # noqa: E402
from inputs import configs as C  # noqa: E402


def main():
    P.load()
    ctx = P.ppca_ctx_create(0, torch.cuda.current_stream())
    # C3-like, d = 1024 (two 512-column slices in the pair kernel, 4 d-groups in the row-group kernel), split
    # layout; ≥ 32768 rows, so the power pass is not the precise (small-shard) variant
    w = dataclasses.replace(C.C3, spec=dataclasses.replace(C.C3.spec, n=40_011))
    s = w.spec
    X = torch.empty((s.n, s.d), dtype=torch.float32, device="cuda")
    P.ppca_generate(ctx, P.gen_spec(s, split=True), X)
    Xm = P.matrix(X, split=True)
    W = torch.empty((w.m, s.d), dtype=torch.float32, device="cuda")
    for impl, kern in ((0, 4), (4, 3), (3, 2)):             # pair kernel, row-group kernel, two kernels
        P.ppca_set_pass_impl(ctx, impl)
        P.ppca_prime_power(ctx, Xm, w.m, 2, w.init_seed, W, theta_hist=True)
        assert P.ppca_last_power_kernel(ctx) == kern, (impl, P.ppca_last_power_kernel(ctx))
    P.ppca_set_pass_impl(ctx, 0)
    E = torch.empty((w.k, s.d), dtype=torch.float32, device="cuda")
    P.ppca_refine(ctx, Xm, W, w.m, w.k, E)
    P.ppca_refine_sampled(ctx, Xm, W, w.m, w.k, E, 0.3, 5)
    # C2-like Oja (the persistent cooperative kernel) and EigenGame window steps
    w2 = dataclasses.replace(C.C2, spec=dataclasses.replace(C.C2.spec, n=4_096))
    s2 = w2.spec
    X2 = torch.empty((s2.n, s2.d), dtype=torch.float32, device="cuda")
    P.ppca_generate(ctx, P.gen_spec(s2, split=True), X2)
    X2m = P.matrix(X2, split=True)
    V = torch.empty((w2.m, s2.d), dtype=torch.float32, device="cuda")
    vel = torch.zeros_like(V)
    P.ppca_prime_oja(ctx, X2m, w2.m, w2.batch, w2.alpha, 0.9, 4, w2.init_seed, V, vel, 0)
    P.ppca_set_pass_impl(ctx, 2)
    P.ppca_prime_eigengame(ctx, X2m, w2.m, w2.batch, 1e-4, 0.9, 2, w2.init_seed, V, vel, 0)
    P.ppca_set_pass_impl(ctx, 0)
    # bf16, m = 128 (2-CTA kernel A2, lean kernel B, blocked Cholesky)
    w5 = dataclasses.replace(C.C5, spec=dataclasses.replace(C.C5.spec, n=12_000, d=2048))
    s5 = w5.spec
    X5 = torch.empty((s5.n, s5.d), dtype=torch.bfloat16, device="cuda")
    P.ppca_generate(ctx, P.gen_spec(s5), X5)
    X5m = P.matrix(X5)
    W5 = torch.empty((w5.m, s5.d), dtype=torch.float32, device="cuda")
    P.ppca_set_pass_impl(ctx, 2)
    P.ppca_prime_power(ctx, X5m, w5.m, 2, w5.init_seed, W5, theta_hist=True)
    E5 = torch.empty((w5.k, s5.d), dtype=torch.float32, device="cuda")
    P.ppca_refine(ctx, X5m, W5, w5.m, w5.k, E5)
    P.ppca_set_pass_impl(ctx, 0)
    torch.cuda.synchronize()
    P.ppca_ctx_destroy(ctx)
    print("sanitize_run: ok")


if __name__ == "__main__":
    main()
