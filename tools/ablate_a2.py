"""Kernel A2 ablation on C5 (experiment build, PPCA_DBG bits of kernel A2: 1 no MMAs, 32 no W' loads): time the
refine pass (kernel A2 alone) on an orthonormal random basis; numerical results are ignored (a skipped load
or MMA leaves garbage, so the Ritz solve may report an error after the timed kernel).

    PPCA_EXP_LIB=paper_2109_03709_b200/libppca_exp.so PPCA_DBG=32 python tools/ablate_a2.py [C5] [reps]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2109_03709_b200 as P  # noqa: E402
from inputs import configs as C  # noqa: E402

if os.environ.get("PPCA_EXP_LIB"):
    P.load(os.environ["PPCA_EXP_LIB"])
name = sys.argv[1] if len(sys.argv) > 1 else "C5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
w = C.FULL[name]
s = w.spec
ctx = P.ppca_ctx_create(0, torch.cuda.current_stream())
dt = torch.float32 if s.dtype == "f32" else torch.bfloat16
X = torch.empty((s.n, s.d), dtype=dt, device="cuda")
P.ppca_generate(ctx, P.gen_spec(s, split=s.dtype == "f32"), X)
Xm = P.matrix(X, split=s.dtype == "f32")
W = torch.linalg.qr(torch.randn(s.d, w.m, device="cuda", dtype=torch.float64))[0].T.contiguous().float()
E = torch.empty((w.k, s.d), device="cuda")
P.ppca_set_timing(ctx, True)
tot, n = 0.0, 0
for r in range(reps + 1):
    P.ppca_get_kernel_time(ctx, 0)
    try:
        P.ppca_refine_ex(ctx, Xm, W, w.m, w.k, E, 1)
    except Exception as e:  # noqa: BLE001 - garbage numerics under the ablation
        pass
    ms, k = P.ppca_get_kernel_time(ctx, 0)
    if r > 0:
        tot += ms
        n += k
gb = s.n * s.d * (4 if s.dtype == "f32" else 2) / 1e9
print(f"{name} kernel A2 (refine pass): {tot / max(n, 1):.3f} ms/launch ({gb / (tot / max(n, 1)) * 1e3:.0f} GB/s), "
      f"PPCA_DBG={os.environ.get('PPCA_DBG', '0')}")
