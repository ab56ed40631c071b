"""C3 pair-kernel pass time vs the number of 2-CTA clusters (experiment build: PPCA_PAIR_NRG caps it).
Prints ppca_get_kernel_time of the pass kernel for 10 power iterations without the θ history."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2109_03709_b200 as P  # noqa: E402
from inputs import configs as C  # noqa: E402
P.load(os.environ.get("PPCA_EXP_LIB", "paper_2109_03709_b200/libppca_exp.so"))
w = C.FULL["C3"]; s = w.spec
ctx = P.ppca_ctx_create(0, torch.cuda.current_stream())
X = torch.empty((s.n, s.d), dtype=torch.float32, device="cuda")
P.ppca_generate(ctx, P.gen_spec(s, split=True), X)
Xm = P.matrix(X, split=True)
W = torch.empty((w.m, s.d), device="cuda")
P.ppca_prime_power(ctx, Xm, w.m, 2, w.init_seed, W)
for hist in (False, True):
    P.ppca_set_timing(ctx, True)
    P.ppca_get_pass_time(ctx); P.ppca_get_kernel_time(ctx, 0)
    P.ppca_prime_power(ctx, Xm, w.m, 10, 0, W, theta_hist=hist)
    kms, kn = P.ppca_get_kernel_time(ctx, 0)
    P.ppca_set_timing(ctx, False)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); P.ppca_prime_power(ctx, Xm, w.m, 10, 0, W, theta_hist=hist); e1.record(); torch.cuda.synchronize()
    print(f"nrg cap {os.environ.get('PPCA_PAIR_NRG', '0')} hist {hist}: pass kernel {kms / max(kn, 1) * 1e3:.1f} us, "
          f"step {e0.elapsed_time(e1) / 10 * 1e3:.1f} us", flush=True)
P.ppca_ctx_destroy(ctx)
