#!/usr/bin/env python
"""bench.py — X-pass HBM throughput and pPCA time-to-LCES (BASELINE.json metric) on B200.

Workload (N=1 default): C3 = BASELINE.json configs[2] (n=10^6, d=1024, fp32, planted λ_j=e^{-j/20},
k=32, l=32, block-power priming), rows sharded contiguously over the ranks.  One step = one power
iteration through the C ABI: the streaming pass over X (Y = XWᵀ, Z = YᵀX, S = YᵀY), the NCCL
all-reduce of [Z|S] (N>1), CholQR2 re-orthonormalisation, and the fp64 Rayleigh–Ritz solve of S
(pPCA of the current iterate).  value = X bytes streamed per step over all ranks ÷ step time.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "X-pass HBM GB/s (% of peak) and pPCA time-to-LCES at 1/2/4/8 B200"
LCES_TARGET = {"C1": math.pi / 1024, "C3": math.pi / 1024, "C5": math.pi / 8}   # reading R20
CFG_INDEX = {"C1": 0, "C2": 1, "C3": 2, "C4": 3, "C5": 4}
DESCR = {"C1": "tiny planted exp spectrum", "C2": "image-like sparse factor model", "C4": "power-law spectrum", "C3": "planted exp spectrum λ_j=e^(-j/20)",
         "C5": "wide activation-like (Householder r=8, ReLU, λ_j=1/j)"}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _traffic(config, impl):
    """Per-launch dram bytes of the pass kernel from a committed ncu --set full summary, if any."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)
        return t.get(f"{config}:{impl}")
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) != 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- CPU oracle legs
def _oracle_sample(w, rows: int):
    """A bounded row sample of the workload for the CPU oracle (raw rows centred by the sample mean)."""
    from inputs import generate as G
    raw = G.raw_rows(w.spec, np.arange(rows))
    x = raw - raw.mean(axis=0, keepdims=True)
    return G.stored_to_f64(G.store(x, w.spec.dtype), w.spec.dtype)


def oracle_step_rate(w, rows: int, steps: int, warmup: int = 0):
    """Time the fp64 oracle's power step (+ Rayleigh–Ritz of S) on `rows` rows; GB/s of stored X."""
    from inputs import generate as G
    from oracle import ppca_oracle as O
    X = _oracle_sample(w, rows)
    W = O.gram_schmidt(O.init_vectors(G.init_gaussians(w.init_seed, w.m, w.spec.d)), drop=False)
    for _ in range(warmup):
        W, S = O.power_step(X, W)
    t0 = time.perf_counter()
    for _ in range(steps):
        W, S = O.power_step(X, W)
        np.linalg.eigvalsh(S)      # the m×m solve (negligible; LAPACK so the timing is the pass)
    dt = (time.perf_counter() - t0) / steps
    nbytes = rows * w.spec.d * (4 if w.spec.dtype == "f32" else 2)
    return nbytes / dt / 1e9, dt


def run_reference(args, w, rank):
    if rank != 0:
        return 0
    rows = args.ref_rows or min(w.spec.n, 65536, (1 << 30) // (8 * w.spec.d))
    gbs, dt = oracle_step_rate(w, rows, max(1, args.steps), max(0, min(args.warmup, 1)))
    cores = os.cpu_count()
    sample = f"{rows} of {w.spec.n} rows of {w.name}; fp64 numpy oracle power step (Y=XWᵀ, Z=YᵀX, S=YᵀY, GS) + eig(S)"
    line = {"impl": "reference", "metric": METRIC, "value": gbs, "unit": "GB/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": w.name, "n": w.spec.n, "d": w.spec.d, "m": w.m, "k": w.k, "priming": w.priming},
            "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def _bf16_peak(sustained=False):
    """Measured dense bf16 TFLOP/s (MEASURED_PEAKS.json): the burst figure, or the sustained one (a kernel timed
    inside a long step); the guide's nominal 2250 if the file is absent."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["bf16_tflops_sustained" if sustained and "bf16_tflops_sustained" in pk else "bf16_tflops"])
    except Exception:
        return 2250.0


def _timed_prime_refine(P, ctx, Xm, w, iters, W, E, stream, barrier, max_over_ranks):
    """ONE timed region: priming from the seeded start (init + `iters` power iterations) and the pPCA refine,
    through the C ABI, CUDA events on the library stream, max over ranks."""
    import torch
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    P.ppca_prime_power(ctx, Xm, w.m, iters, w.init_seed, W)
    P.ppca_refine_ex(ctx, Xm, W, w.m, w.k, E, P.PPCA_REFINE_ORTHONORMAL)     # W is orthonormal (CholQR)
    e1.record(stream)
    torch.cuda.synchronize()
    return {"ms": max_over_ranks(e0.elapsed_time(e1)), "timed": "init + power iterations + refine, one region"}


def time_to_subspace_target(P, ctx, Xm, w, s, dev, stream, max_over_ranks, target=1e-2):
    """C5 (reading R20): iterations until the pPCA top-k subspace error ≤ 1e-2 against a residual-certified
    reference (reading R29): 80 power iterations + refine from an independent start, its Ritz
    pairs certified by one exact-fp32 residual pass (Weyl: |λ − θ| ≤ r; Davis–Kahan: sinΘ ≤ ‖R_k‖_F / δ,
    δ = θ_k − (θ_{k+1} + r_{k+1})).  Evaluation is untimed; the run to the target is then timed end to end."""
    import torch
    k1 = w.k + 1
    Wr = torch.empty((w.m, s.d), dtype=torch.float32, device=dev)
    # the reference: 60 tensor-core iterations, then 16 on the exact-fp32 CUDA-core pass (its span is not held
    # back by the bf16 rounding of Y in product 2, R27) and a CUDA-core refine
    P.ppca_prime_power(ctx, Xm, w.m, 60, w.init_seed + 7919, Wr)
    P.ppca_set_pass_impl(ctx, 1)
    try:
        P.ppca_prime_power(ctx, Xm, w.m, 16, 0, Wr)
        Eref = torch.empty((k1, s.d), dtype=torch.float32, device=dev)
        th_ref, _ = P.ppca_refine(ctx, Xm, Wr, w.m, k1, Eref)
    finally:
        P.ppca_set_pass_impl(ctx, 0)
    res, rgram = P.ppca_ritz_residuals(ctx, Xm, Eref, k1, th_ref, gram=True)
    delta = th_ref[w.k - 1] - (th_ref[w.k] + res[w.k])
    r2 = float(np.sqrt(max(0.0, np.linalg.eigvalsh(rgram[: w.k, : w.k])[-1])))      # ‖R_k‖₂
    bound = r2 / delta if delta > 0 else float("inf")
    T = Eref[: w.k].double()

    def sub_err(E):
        A = E.double() - (E.double() @ T.T) @ T
        return float(torch.linalg.svdvals(A)[0])

    W2 = torch.empty_like(Wr)
    E = torch.empty((w.k, s.d), dtype=torch.float32, device=dev)
    P.ppca_prime_power(ctx, Xm, w.m, 0, w.init_seed, W2)
    reached, measured, errs = None, None, []
    for t in range(1, w.iters + 1):
        P.ppca_prime_power(ctx, Xm, w.m, 1, 0, W2)
        P.ppca_refine_ex(ctx, Xm, W2, w.m, w.k, E, P.PPCA_REFINE_ORTHONORMAL)
        errs.append(sub_err(E))
        if measured is None and errs[-1] <= target:
            measured = t
        if errs[-1] + bound <= target:                # certified: the error to the TRUE subspace is ≤ target
            reached = t
            break
    out = {"target": f"top-{w.k} subspace error <= {target} to the true subspace (measured error vs the reference "
                     f"+ the reference's certified bound)",
           "iterations": reached, "iterations_measured_only": measured, "subspace_error_per_iteration": errs,
           "reference": {"iterations": "60 tensor-core + 16 exact-fp32", "theta_1": float(th_ref[0]),
                         "max_residual_over_theta1":
                         float(np.max(res[: w.k]) / th_ref[0]), "certified_subspace_bound": bound,
                         "how": "power + refine from an independent start; ppca_ritz_residuals (exact-fp32 pass)"}}
    out["certified"] = reached is not None
    if reached:
        def nob():
            pass
        out.update(_timed_prime_refine(P, ctx, Xm, w, reached, W2, E, stream, nob, max_over_ranks))
        out["subspace_error_at_end_of_timed_run"] = sub_err(E)
    return out


# ----------------------------------------------------------------------------- GPU arm
def run_ours(args, w, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    import paper_2109_03709_b200 as P

    P.load()
    assert not P.ppca_experiments_enabled(), "libppca.so built with -DPPCA_EXPERIMENTS: not a product build"
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    stream = torch.cuda.current_stream()
    ctx = P.ppca_ctx_create_distributed(local_rank, stream)
    impl_code = {"auto": 0, "simt": 1, "tc": 2}[args.pass_impl]
    P.ppca_set_pass_impl(ctx, impl_code)
    s = w.spec
    per = -(-s.n // world)
    _, n_local = P.contiguous_shard(s.n, rank, world)
    dt = torch.float32 if s.dtype == "f32" else torch.bfloat16
    elt = 4 if s.dtype == "f32" else 2
    X = torch.empty((max(n_local, 1), s.d), dtype=dt, device=dev)[:n_local]
    t0 = time.time()
    P.ppca_generate(ctx, P.gen_spec(s), X if n_local else torch.empty((0, s.d), dtype=dt, device=dev))
    torch.cuda.synchronize()
    gen_s = time.time() - t0
    # fp32 data is held in the tensor-core-native split layout (include/ppca.h PPCA_F32_SPLIT): same bytes
    split = s.dtype == "f32" and args.storage == "split"
    Xh = None
    if split:
        if not args.no_e2e and n_local > 0:
            Xh = torch.empty(X.shape, dtype=dt, pin_memory=True)      # the user's fp32 rows, for e2e
            Xh.copy_(X)
        P.ppca_split_f32(ctx, X, s.d)
    Xm = P.matrix(X, n_global=s.n, d=s.d, split=split)
    W = torch.empty((w.m, s.d), dtype=torch.float32, device=dev)
    P.ppca_prime_power(ctx, Xm, w.m, 0, w.init_seed, W)             # W_0
    P.ppca_prime_power(ctx, Xm, w.m, args.warmup, 0, W, theta_hist=True)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---------------- kernel timing: an instrumented region (CUDA events around the pass kernels on the library
    # stream) of the same K steps; the events would break the programmatic dependent launches of the chain, so
    # the step time (value) comes from the uninstrumented timed region below
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    P.ppca_set_timing(ctx, True)
    P.ppca_get_pass_time(ctx)
    P.ppca_get_kernel_time(ctx, 0), P.ppca_get_kernel_time(ctx, 1)
    barrier()
    torch.cuda.synchronize()
    ev0.record(stream)
    P.ppca_prime_power(ctx, Xm, w.m, args.steps, 0, W, theta_hist=True)
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms_prof = max_over_ranks(ev0.elapsed_time(ev1))
    pass_ms_tot, passes = P.ppca_get_pass_time(ctx)
    ka_ms_tot, ka_n = P.ppca_get_kernel_time(ctx, 0)      # kernel A: Y = X·W'ᵀ, S = YᵀY (reads X once)
    kb_ms_tot, kb_n = P.ppca_get_kernel_time(ctx, 1)      # kernel B: Zᵀ = X_hiᵀ·Y
    P.ppca_set_timing(ctx, False)
    # ---------------- timed region (inputs 4 GB ≫ 126 MB L2: no flush needed)
    l0 = P.ppca_launch_count(ctx)
    k0 = P.ppca_collective_count(ctx)
    with ClockSampler(local_rank) as clk:
        barrier()
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_push("timed")
        ev0.record(stream)
        P.ppca_prime_power(ctx, Xm, w.m, args.steps, 0, W, theta_hist=True)
        ev1.record(stream)
        torch.cuda.nvtx.range_pop()
        torch.cuda.synchronize()
        barrier()
    launches = P.ppca_launch_count(ctx) - l0
    collectives = P.ppca_collective_count(ctx) - k0
    ms = max_over_ranks(ev0.elapsed_time(ev1))
    ms_step = ms / args.steps
    bytes_step = s.n * s.d * elt                       # whole job: every rank streams its shard once
    value = bytes_step * args.steps / (ms / 1e3) / 1e9
    pass_ms = max_over_ranks(pass_ms_tot / max(passes, 1))
    per_rank_bytes = per * s.d * elt
    peak, peak_src = _peaks()
    pass_achieved = per_rank_bytes / (pass_ms / 1e3) / 1e9
    plan_impl = {1: "simt", 2: "tcgen05"}.get(P.ppca_last_pass_impl(ctx), "none")
    # roofline of the dominant kernel (largest device time in the timed region): algorithmic bytes per
    # launch = the X bytes that kernel must read (kernel A: all of X; kernel B: the X_hi plane of a split
    # X, the bf16 X, or the fp32 X) ÷ its average launch time (CUDA events on the library stream)
    kb_elt = 2 if (split or s.dtype == "bf16") else 4
    kernels = []
    if ka_n and not kb_n:                              # the single-read fused power pass (one kernel)
        fk = ("xwz_pair_kernel (single-read power pass on d-sliced CTA pairs: Y = X W'^T, S = Y^T Y, Z^T = X^T Y)"
              if P.ppca_last_power_kernel(ctx) == 4 else
              "xwz_fused_kernel (single-read power pass, row groups: Y = X W'^T, S = Y^T Y, Z^T = X^T Y)")
        kernels.append((fk, ka_ms_tot, ka_n, per_rank_bytes))
    elif ka_n:
        kernels.append(("xw_tma_kernel (kernel A2: Y = X W'^T, S = Y^T Y)" if s.dtype != "f32" or split
                        else "xw_tc_kernel (kernel A: Y = X W'^T, S = Y^T Y)", ka_ms_tot, ka_n, per_rank_bytes))
    if kb_n:
        kernels.append(("xty_tc_kernel (kernel B: Z^T = X_hi^T Y)", kb_ms_tot, kb_n, per * s.d * kb_elt))
    if kernels and len(kernels) == 1:                  # the single-read fused kernel is the pass
        kname, k_tot, k_n, k_bytes = kernels[0]
        k_ms = max_over_ranks(k_tot / k_n)
        kernel_share = k_tot / max(ms_prof, 1e-9)
    else:                                              # two kernels (X read twice) or SIMT: the whole pass, vs
        kname = (f"power pass ({' + '.join(k[0].split()[0] for k in kernels)} + reductions; X read twice)"
                 if kernels else f"streaming pass ({plan_impl})")
        k_ms, k_n, k_bytes = pass_ms, passes, per_rank_bytes          # ONE read of X (algorithmic bytes)
        kernel_share = pass_ms_tot / max(ms_prof, 1e-9)
    achieved = k_bytes / (k_ms / 1e3) / 1e9
    # the contraction's own roofline (context): algorithmic 4·n·d·m flop per power pass against the measured
    # bf16 dense peak (burst: the kernels are timed inside the step's sequence, not back to back for seconds)
    flops_pass = 4.0 * per * s.d * w.m
    # executed MMA work: product 1 X·[W_hi;W_lo]^T (N = 2m) + X_lo·W_hi^T (N = m, split X); product 2 X_hi^T·Y with
    # Y_hi alone (N = m, bf16 X outside the fused kernels: R27) or [Y_hi; Y_lo] (N = 2m); S = YᵀY is negligible
    lean_p2 = s.dtype == "bf16" and kernels and len(kernels) == 2
    n_p1 = 2 * w.m + (w.m if split else 0)
    n_p2 = w.m if lean_p2 else 2 * w.m
    exec_flops = 2.0 * per * s.d * (n_p1 + n_p2)
    sus = _bf16_peak(sustained=True)
    tensor_ctx = {"algorithmic_tflop_per_pass": flops_pass / 1e12, "achieved_tflops": flops_pass / (pass_ms / 1e3) / 1e12,
                  "peak_tflops": _bf16_peak(), "frac": flops_pass / (pass_ms / 1e3) / 1e12 / _bf16_peak(),
                  "executed_tflop_per_pass": exec_flops / 1e12,
                  "executed_tflops": exec_flops / (pass_ms / 1e3) / 1e12,
                  "sustained_peak_tflops": sus,
                  "executed_frac_of_sustained": exec_flops / (pass_ms / 1e3) / 1e12 / sus,
                  "executed_mma_note": "product 1 runs X·[W_hi;W_lo]^T (N = 2m) for the fp32-accurate operand (DESIGN "
                                       "R27), plus X_lo·W_hi^T for a split X; executed_frac_of_sustained is the pass "
                                       "against the measured sustained bf16 peak (it runs inside a long step)"}

    # ---------------- end to end through the ABI with host buffers (H2D of X + D2H of θ every step)
    e2e = None
    if not args.no_e2e and n_local > 0:
        if Xh is None:
            Xh = torch.empty(X.shape, dtype=dt, pin_memory=True)
            Xh.copy_(X)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ke = max(1, min(args.steps, 5))
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(ke):
            P.ppca_upload_rows(ctx, Xh, Xm)                               # the user's rows, host → HBM (+ split)
            P.ppca_prime_power(ctx, Xm, w.m, 1, 0, W, theta_hist=True)   # θ read back to the host
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ems = max_over_ranks(e0.elapsed_time(e1))
        e2e = {"value": bytes_step * ke / (ems / 1e3) / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": int(bytes_step), "d2h_bytes_per_step": int(8 * w.m * world)}
        del Xh

    # ---------------- time to LCES (reading R20): find the iteration untimed, then time the whole
    # priming-from-the-seed + refine in ONE region (CUDA events on the library stream)
    ttl = None
    if not args.no_lces and s.d > 4096:
        ttl = time_to_subspace_target(P, ctx, Xm, w, s, dev, stream, max_over_ranks)
    if not args.no_lces and s.d <= 4096:
        G64 = torch.zeros((s.d, s.d), dtype=torch.float64, device=dev)
        P.ppca_gram(ctx, Xm, G64)
        lam, U = np.linalg.eigh(G64.cpu().numpy())
        T = U[:, ::-1][:, : w.k].T.copy()
        Tt = torch.from_numpy(T.astype(np.float32)).to(dev)
        thr = LCES_TARGET.get(w.name, math.pi / 8)
        W2 = torch.empty_like(W)
        E = torch.empty((w.k, s.d), dtype=torch.float32, device=dev)
        P.ppca_prime_power(ctx, Xm, w.m, 0, w.init_seed, W2)
        reached = None
        for t in range(1, w.iters + 1):
            P.ppca_prime_power(ctx, Xm, w.m, 1, 0, W2)
            P.ppca_refine(ctx, Xm, W2, w.m, w.k, E)
            _, lc = P.ppca_eval(ctx, E, Tt, w.k, s.d, [thr])
            if lc[0] >= w.k:
                reached = t
                break
        r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        r0.record(stream)
        P.ppca_refine(ctx, Xm, W2, w.m, w.k, E)
        r1.record(stream)
        torch.cuda.synchronize()
        refine_ms = max_over_ranks(r0.elapsed_time(r1))
        ttl = {"target": f"LCES={w.k} at V={thr:.6f}", "iterations": reached, "refine_ms": refine_ms}
        if reached:
            ttl.update(_timed_prime_refine(P, ctx, Xm, w, reached, W2, E, stream, barrier, max_over_ranks))
            _, lc = P.ppca_eval(ctx, E, Tt, w.k, s.d, [thr])
            ttl["lces_at_end_of_timed_run"] = int(lc[0])

    P.ppca_ctx_destroy(ctx)
    del X, Xm, W

    if rank != 0:
        return None
    cpu = None
    if world == 1 and not args.no_cpu:
        rows = args.cpu_rows or min(s.n, 131072, (1 << 30) // (8 * s.d))   # ≤ 1 GiB of fp64 sample
        gbs, dt_s = oracle_step_rate(w, rows, 2, 0)
        cpu = {"value": gbs, "unit": "GB/s", "cores": os.cpu_count(), "kind": "oracle",
               "sample": f"{rows} of {s.n} rows of {w.name}, 2 fp64 numpy oracle power steps "
                         f"({dt_s * 1e3:.0f} ms/step); X bytes counted at the stored {s.dtype}"}
    clocks = clk.summary()
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": s.dtype, "data": "synthetic",
        "config": {"workload": f"{w.name} (BASELINE.json configs[{CFG_INDEX.get(w.name, '?')}]): {DESCR.get(w.name, '')}, "
                               f"n={s.n}, d={s.d}, {s.dtype}, k={w.k}, l={w.l}, block power priming",
                   "n": s.n, "d": s.d, "m": w.m, "k": w.k, "priming": w.priming, "pass_impl": plan_impl,
                   "storage": "f32 split (bf16 hi/lo planes, 4 B/elt)" if split else s.dtype,
                   "parallelism": f"dp{world} (contiguous row shards, NCCL all-reduce of Z,S)",
                   "l2": f"inputs larger than L2 (X shard {per_rank_bytes / 1e9:.2f} GB vs 126 MB L2)",
                   "step": "pass + allreduce + CholQR2 + fp64 Rayleigh-Ritz of S"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": _traffic(w.name, kname.split()[0]),
                     "kernel": kname, "kernel_ms": k_ms, "launches": k_n, "share_of_timed_region": kernel_share,
                     "algorithmic_bytes_per_launch": k_bytes, "peak_source": peak_src,
                     "pass": {"ms": pass_ms, "achieved": pass_achieved, "frac": pass_achieved / peak,
                              "note": "whole power pass (all its kernels + reductions) vs one read of X"},
                     "tensor_context": tensor_ctx},
        "step_outside_pass_ms": ms_step - pass_ms,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "nccl_collectives": int(collectives),
        "clocks": clocks,
        "time_to_lces": ttl,
        "generate_s": gen_s,
    }
    return line


# ----------------------------------------------------------------------------- minibatch primings (C2, C4)
def oracle_minibatch_rate(w, rows: int, steps: int):
    """The fp64 oracle's minibatch step (Oja / EigenGame) on the first `rows` rows; GB/s of stored X."""
    from inputs import generate as G
    from oracle import ppca_oracle as O
    X = _oracle_sample(w, rows)
    V = O.init_vectors(G.init_gaussians(w.init_seed, w.m, w.spec.d))
    vel = np.zeros_like(V)
    step = O.oja_step if w.priming == "oja" else O.eigengame_step
    b = min(w.batch, rows)
    t0 = time.perf_counter()
    for k in range(steps):
        r0 = (k * b) % max(1, rows - b + 1)
        V, vel = step(X[r0:r0 + b], V, vel, w.alpha, w.momentum)
    dt = (time.perf_counter() - t0) / steps
    return b * w.spec.d * 4 / dt / 1e9, dt


def run_minibatch(args, w, rank, world, local_rank):
    """One step = one minibatch priming step (P L70-72 generalized Oja, or P L76-88 EigenGame) over the
    global batch: the window pass (Y = X_b·W'ᵀ, Q = X_bᵀY, P = YᵀY), the all-reduce (N>1) and the update.
    value = X bytes of the global batch per step ÷ step time (the batch is re-read every step)."""
    import torch
    import torch.distributed as dist
    import paper_2109_03709_b200 as P
    P.load()
    assert not P.ppca_experiments_enabled(), "libppca.so built with -DPPCA_EXPERIMENTS: not a product build"
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    stream = torch.cuda.current_stream()
    ctx = P.ppca_ctx_create_distributed(local_rank, stream)
    P.ppca_set_pass_impl(ctx, {"auto": 0, "simt": 1, "tc": 2}[args.pass_impl])
    s = w.spec
    split = s.dtype == "f32" and args.storage == "split"
    layout = P.PPCA_LAYOUT_INTERLEAVED if world > 1 else P.PPCA_LAYOUT_CONTIGUOUS
    from inputs import generate as G
    n_local = len(G.shard_rows(s.n, rank, world, "interleaved" if world > 1 else "contiguous", w.batch))
    X = torch.empty((max(n_local, 1), s.d), dtype=torch.float32, device=dev)[:n_local]
    P.ppca_generate(ctx, P.gen_spec(s, layout=layout, block_rows=w.batch if world > 1 else 0, split=split), X)
    Xm = P.matrix(X, n_global=s.n, d=s.d, split=split, layout=layout, block_rows=w.batch if world > 1 else 0)
    fn = P.ppca_prime_oja if w.priming == "oja" else P.ppca_prime_eigengame
    V = torch.empty((w.m, s.d), dtype=torch.float32, device=dev)
    vel = torch.zeros_like(V)
    steps = max(args.steps, 1) * (20 if w.priming == "oja" else 5)     # ≥ 50 steps (µs-scale steps)
    step0 = fn(ctx, Xm, w.m, w.batch, w.alpha, w.momentum, max(args.warmup, 3), w.init_seed, V, vel, 0)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # kernel times from an instrumented run of the same steps (the events around the window-pass kernels break
    # the programmatic dependent launches of the step: ≈ 25 µs per C4 step), the step time uninstrumented
    P.ppca_set_timing(ctx, True)
    P.ppca_get_pass_time(ctx), P.ppca_get_kernel_time(ctx, 0), P.ppca_get_kernel_time(ctx, 1)
    step0 = fn(ctx, Xm, w.m, w.batch, w.alpha, w.momentum, steps, 0, V, vel, step0)
    torch.cuda.synchronize()
    pass_ms_tot, passes = P.ppca_get_pass_time(ctx)
    ka_ms, ka_n = P.ppca_get_kernel_time(ctx, 0)
    kb_ms, kb_n = P.ppca_get_kernel_time(ctx, 1)
    P.ppca_set_timing(ctx, False)
    l0 = P.ppca_launch_count(ctx)
    with ClockSampler(local_rank) as clk:
        barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        fn(ctx, Xm, w.m, w.batch, w.alpha, w.momentum, steps, 0, V, vel, step0)
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
    launches = P.ppca_launch_count(ctx) - l0
    ms = max_over_ranks(ev0.elapsed_time(ev1))
    ms_step = ms / steps
    batch_bytes = w.batch * s.d * 4
    value = batch_bytes / (ms_step / 1e3) / 1e9
    peak, peak_src = _peaks()
    local_batch = w.batch // world
    if ka_n or kb_n:       # the tensor-core window pass: kernel A2 (K-split) and the precise kernel B
        cand = [("xw_tma_kernel (kernel A2, K-split over the step's window)", ka_ms, ka_n),
                ("xty_tc_kernel (kernel B, X_hi and X_lo planes)", kb_ms, kb_n)]
        kname, k_tot, k_n = max(cand, key=lambda k: k[1])
        k_ms = max_over_ranks(k_tot / max(k_n, 1))
        k_bytes = local_batch * s.d * 4
    elif launches == 1:    # short windows on one GPU: every step inside one cooperative kernel
        kname, k_ms, k_n, k_bytes = "oja_persistent_kernel (all steps in one cooperative launch; grid-barrier " \
            "latency bound)", ms_step, steps, local_batch * s.d * 4
    else:                  # small windows run the CUDA-core kernels: the whole (launch-bound) step is reported
        kname, k_ms, k_n, k_bytes = "minibatch step (CUDA-core window kernels; launch-latency bound)", ms_step, \
            steps, local_batch * s.d * 4
    achieved = k_bytes / (k_ms / 1e3) / 1e9
    ttl = None
    if not args.no_lces and world == 1 and s.d <= 4096:
        G64 = torch.zeros((s.d, s.d), dtype=torch.float64, device=dev)
        P.ppca_gram(ctx, P.matrix(X, split=split), G64)
        lam, U = np.linalg.eigh(G64.cpu().numpy())
        del G64
        Tt = torch.from_numpy(U[:, ::-1][:, : w.k].T.copy().astype(np.float32)).to(dev)
        thr = math.pi / 8                               # reading R20 for the minibatch configs
        V2 = torch.empty_like(V)
        vel2 = torch.zeros_like(V)
        E = torch.empty((w.k, s.d), dtype=torch.float32, device=dev)
        per_epoch = -(-s.n // w.batch)
        checkpoints = sorted(set([2 ** j for j in range(4, 13)] + [per_epoch * e for e in range(1, 31)]))
        cap = 30 * per_epoch if w.priming == "oja" else 4096       # reading R21
        def ttl_run(fraction):
            """priming from the seeded start, a charged refine at every checkpoint until LCES = k; fraction < 1:
            the refine projects a seeded 10 % row-tile sample (P L378, reading R25)"""
            def refine():
                if fraction >= 1.0:
                    P.ppca_refine(ctx, Xm, V2, w.m, w.k, E)
                else:
                    P.ppca_refine_sampled(ctx, Xm, V2, w.m, w.k, E, fraction, 4242)
            vel2.zero_()
            step = fn(ctx, Xm, w.m, w.batch, w.alpha, w.momentum, 0, w.init_seed, V2, vel2, 0)
            refine()                                     # untimed warm-up: the refine's scratch and kernels
            torch.cuda.synchronize()
            step = fn(ctx, Xm, w.m, w.batch, w.alpha, w.momentum, 0, w.init_seed, V2, vel2, 0)
            reached, t_ms = None, 0.0
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            for cp in checkpoints:
                if cp > cap:
                    break
                e0.record(stream)
                step = fn(ctx, Xm, w.m, w.batch, w.alpha, w.momentum, cp - step, 0, V2, vel2, step)
                refine()                                 # charged refine (S L429)
                e1.record(stream)
                torch.cuda.synchronize()
                t_ms += e0.elapsed_time(e1)
                _, lc = P.ppca_eval(ctx, E, Tt, w.k, s.d, [thr])
                if lc[0] >= w.k:
                    reached = cp
                    break
            return reached, t_ms

        reached, t_ms = ttl_run(1.0)
        ttl = {"target": f"LCES={w.k} at V={thr:.6f}", "steps": reached,
               "ms": t_ms if reached else None, "checkpoints": "2^j and every epoch, refine charged",
               "refine": "full projection"}
        if s.n >= 1_000_000:                             # the paper's large-n setting: project 10 % (P L378)
            r2, t2 = ttl_run(0.1)
            ttl["sampled_refine"] = {"steps": r2, "ms": t2 if r2 else None,
                                     "refine": "seeded 10 % row-tile sample (P L378, reading R25)"}
    P.ppca_ctx_destroy(ctx)
    if rank != 0:
        return 0
    cpu = None
    if world == 1 and not args.no_cpu:
        rows = min(s.n, w.batch * (16 if w.priming == "oja" else 1))    # host generation of the sample is costly
        ksteps = 200 if w.priming == "oja" else 10
        gbs, dt_s = oracle_minibatch_rate(w, rows, ksteps)
        cpu = {"value": gbs, "unit": "GB/s", "cores": os.cpu_count(), "kind": "oracle",
               "sample": f"{ksteps} fp64 numpy oracle {w.priming} steps (batch {min(w.batch, rows)}) on {rows} of "
                         f"{s.n} rows of {w.name} ({dt_s * 1e3:.1f} ms/step)"}
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": s.dtype, "data": "synthetic",
        "config": {"workload": f"{w.name} (BASELINE.json configs[{CFG_INDEX.get(w.name, '?')}]): {w.priming} priming, "
                               f"n={s.n}, d={s.d}, batch={w.batch}, alpha={w.alpha}, momentum={w.momentum}, "
                               f"k={w.k}, l={w.l}",
                   "n": s.n, "d": s.d, "m": w.m, "k": w.k, "priming": w.priming, "batch": w.batch,
                   "storage": "f32 split (bf16 hi/lo planes, 4 B/elt)" if split else s.dtype,
                   "parallelism": f"dp{world} (interleaved block rows, NCCL all-reduce of Q,P per step)",
                   "l2": f"batch {batch_bytes / 1e6:.1f} MB per step re-read from HBM/L2 (X {s.n * s.d * 4 / 1e9:.2f} GB)",
                   "step": "window pass + all-reduce + update (one minibatch step)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": None, "kernel": kname, "kernel_ms": k_ms, "launches": k_n,
                     "algorithmic_bytes_per_launch": k_bytes, "peak_source": peak_src},
        "cpu_baseline": cpu, "e2e": None, "gpu_launches": int(launches), "clocks": clk.summary(),
        "time_to_lces": ttl,
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    from inputs import configs as C
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C3")
    ap.add_argument("--pass-impl", default="auto", choices=["auto", "simt", "tc"])
    ap.add_argument("--storage", default="split", choices=["split", "f32"],
                    help="layout of fp32 X in HBM (split = PPCA_F32_SPLIT, the default)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-lces", action="store_true")
    ap.add_argument("--cpu-rows", type=int, default=0)
    ap.add_argument("--ref-rows", type=int, default=0)
    ap.add_argument("--no-extra", action="store_true", help="skip the C5 (largest config) sub-line of the C3 run")
    args = ap.parse_args()
    w = C.FULL[args.config] if args.config in C.FULL else C.SMALL[args.config]
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        if w.priming != "power":
            raise SystemExit("--impl reference times the power step (C1, C3, C5)")
        return run_reference(args, w, rank)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return _spawn(args)                          # one process per GPU (torchrun), rank 0 prints the line
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    if w.priming == "power":
        line = run_ours(args, w, rank, world, local_rank)
        extra = None
        if args.config == "C3" and not args.no_extra:
            # the largest config (the ≥6× scaling target of BASELINE.json) measured in the same run
            a5 = argparse.Namespace(**vars(args))
            a5.steps, a5.warmup, a5.no_e2e, a5.no_cpu = max(3, min(args.steps, 10)), max(3, args.warmup), True, True
            extra = run_ours(a5, C.FULL["C5"], rank, world, local_rank)
        if rank == 0:
            if extra is not None:
                keep = ["value", "unit", "ms_per_step", "steps", "warmup", "config", "roofline",
                        "step_outside_pass_ms", "gpu_launches", "nccl_collectives", "clocks", "time_to_lces",
                        "generate_s"]
                line["also"] = {"C5": {k: extra[k] for k in keep if k in extra}}
            print(json.dumps(line), flush=True)
        rc = 0
    else:
        rc = run_minibatch(args, w, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return rc


def _spawn(args) -> int:
    """`bench.py --gpus N` without a launcher: re-run this command under torch.distributed.run with N ranks on
    this node (127.0.0.1 rendezvous); the ranks' exit code is returned, rank 0's JSON line is the output."""
    import torch
    n = torch.cuda.device_count()
    if n < args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus}: only {n} CUDA device(s) visible")
    port = 29500 + os.getpid() % 2000
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


if __name__ == "__main__":
    sys.exit(main())
