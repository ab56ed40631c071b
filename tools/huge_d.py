"""the paper's large-scale regime (§5.2) on one B200 with the library's
kernels.  ResNet-152 activations: d ≈ 13.1M, n = 50000, EigenGame batch 1024, k = 8 with no extra components
(L373 "without additional components"), a 10 % row sample for the projection (L378).

Stand-in (no dataset is read): planted Householder + ReLU activations (the C5 family, λ_j = 1/j) in bf16 at
d = 13,107,200.  n = 50000 rows are 1.31 TB of bf16 — 8 B200s hold them row-sharded (164 GB per GPU); this run
is ONE rank's shard (n_local = 6250 rows of the 8-GPU job, contiguous layout), X resident in HBM, the priming
on that shard (batch 1024 rows of it), i.e. exactly the per-GPU work of the 8-GPU run minus the all-reduce.

Reports: EigenGame step time and its X bytes / s; refine (full projection) and sampled refine (10 %) times;
properties that hold at any size (E orthonormal, captured variance of each Ritz vector = θ_i, θ_1 ≥ the best
priming Rayleigh quotient, Ky Fan sums); the parity of these kernel paths against the oracle is
tests/test_gpu_r2.py::test_huge_d_eigengame_and_refine_vs_oracle (d = 524288).

    python tools/huge_d.py [--n 6250] [--d 13107200] [--steps 600] [--out profiles/r2_huge_d.txt]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2109_03709_b200 as P  # noqa: E402
from inputs import generate as G  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=6250)
    ap.add_argument("--d", type=int, default=13_107_200)
    ap.add_argument("--k", type=int, default=8)
    ap.add_argument("--batch", type=int, default=1024)
    ap.add_argument("--steps", type=int, default=600)
    ap.add_argument("--alpha", type=float, default=1e-2)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    P.load()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream()
    ctx = P.ppca_ctx_create(0, stream)
    spec = G.GenSpec("planted_householder", n=a.n, d=a.d, seed=1006, spectrum="power", a=1.0, relu=True, house_r=8,
                     dtype="bf16")
    out = {"workload": f"huge-d stand-in: planted Householder r=8 + ReLU, lambda_j=1/j, bf16, n_local={a.n}, d={a.d} "
                       f"(one rank's shard of 50000 x {a.d} over 8 GPUs), EigenGame batch {a.batch}, k={a.k}, l=0"}
    X = torch.empty((a.n, a.d), dtype=torch.bfloat16, device=dev)
    t0 = time.time()
    P.ppca_generate(ctx, P.gen_spec(spec), X)
    torch.cuda.synchronize()
    out["generate_s"] = time.time() - t0
    out["x_gb"] = a.n * a.d * 2 / 1e9
    Xm = P.matrix(X)
    k = a.k
    V = torch.empty((k, a.d), dtype=torch.float32, device=dev)
    vel = torch.zeros_like(V)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    step = P.ppca_prime_eigengame(ctx, Xm, k, a.batch, a.alpha, 0.9, 3, 2006, V, vel, 0)    # warm-up
    e0.record(stream)
    step = P.ppca_prime_eigengame(ctx, Xm, k, a.batch, a.alpha, 0.9, a.steps - 3, 0, V, vel, step)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / (a.steps - 3)
    out["eigengame_step_ms"] = ms
    out["eigengame_window_gbs"] = a.batch * a.d * 2 / (ms / 1e3) / 1e9
    E = torch.empty((k, a.d), dtype=torch.float32, device=dev)
    th, _ = P.ppca_refine(ctx, Xm, V, k, k, E)                                      # warm-up
    e0.record(stream)
    th, dim = P.ppca_refine(ctx, Xm, V, k, k, E)
    e1.record(stream)
    torch.cuda.synchronize()
    out["refine_ms"] = e0.elapsed_time(e1)
    out["refine_pass_gbs"] = a.n * a.d * 2 / (out["refine_ms"] / 1e3) / 1e9
    Es = torch.empty_like(E)
    P.ppca_refine_sampled(ctx, Xm, V, k, k, Es, 0.1, 4242)
    e0.record(stream)
    ths, _, used = P.ppca_refine_sampled(ctx, Xm, V, k, k, Es, 0.1, 4242)
    e1.record(stream)
    torch.cuda.synchronize()
    out["sampled_refine_ms"] = e0.elapsed_time(e1)
    out["sampled_rows"] = int(used)
    # properties at any size
    Eh = E.double()
    gram = (Eh @ Eh.T).cpu().numpy()
    out["E_orthonormality_err"] = float(np.max(np.abs(gram - np.eye(k))))
    cv = P.ppca_captured_variance(ctx, Xm, E, k)
    out["captured_variance_vs_theta_rel"] = float(np.max(np.abs(cv - th) / th))
    Vn = (V / V.norm(dim=1, keepdim=True)).contiguous()
    rq = P.ppca_captured_variance(ctx, Xm, Vn, k)                                   # priming Rayleigh quotients
    out["theta1_over_best_priming_rq"] = float(th[0] / np.max(rq))
    out["theta"] = [float(x) for x in th]
    out["sampled_theta_rel_diff"] = float(np.max(np.abs(ths - th) / th))
    ok = out["E_orthonormality_err"] < 1e-4 and out["captured_variance_vs_theta_rel"] < 1e-3 and \
        out["theta1_over_best_priming_rq"] >= 1 - 1e-6
    out["properties_hold"] = bool(ok)
    P.ppca_ctx_destroy(ctx)
    txt = json.dumps(out, indent=1)
    print(txt)
    if a.out:
        with open(a.out, "w") as f:
            f.write(txt + "\n")
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
