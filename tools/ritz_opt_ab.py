"""Experiment build: ritz_values_kernel's opt bits (PPCA_RITZ_OPT: 1 product-form Sturm counts, 2 warp-per-row
tridiagonalisation matvec, 4 register-tiled C = L^-1 S L^-T).  One process per setting: phase clocks on C3s,
theta history / refine theta / E saved to /tmp for the comparison (`tools/ritz_opt_ab.py cmp 0 1 2 4 7`)."""
import ctypes, os, sys
import numpy as np
if len(sys.argv) > 1 and sys.argv[1] == "cmp":
    ref = np.load(f"/tmp/ritz_opt_{sys.argv[2]}.npz")
    for o in sys.argv[3:]:
        z = np.load(f"/tmp/ritz_opt_{o}.npz")
        out = []
        for k in ref.files:
            a, b = ref[k], z[k]
            out.append(f"{k} {np.max(np.abs(a - b) / np.maximum(np.abs(a), 1e-300)) if k.startswith('th') else np.max(np.abs(a - b)):.2e}")
        print(f"opt={o} vs opt={sys.argv[2]}: " + "  ".join(out))
    sys.exit(0)
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2109_03709_b200 as P
from inputs import configs as C, generate as G
lib = P.load(os.environ["PPCA_EXP_LIB"]); lib.ppca_debug_wait_counters.argtypes = [ctypes.c_void_p]
opt = os.environ.get("PPCA_RITZ_OPT", "0")
names = ["cholesky", "L^-1", "C=L^-1 S L^-T", "tridiag", "multisection", "inv-iteration", "back-transform"]
def show(tag):
    out = (ctypes.c_ulonglong * 16)(); lib.ppca_debug_wait_counters(out)
    c = [out[i] for i in range(8)]
    print(f"opt={opt}", tag, "  ".join(f"{n} {(c[i+1]-c[i])/1.9e3:.1f}us" for i, n in enumerate(names) if c[i+1] > c[i]), flush=True)
ctx = P.ppca_ctx_create(0, torch.cuda.current_stream())
res = {}
for name in ("C3s", "C1"):
    w = C.SMALL[name] if name in C.SMALL else getattr(C, name); s = w.spec
    X = torch.from_numpy(np.ascontiguousarray(G.dataset(s), dtype=np.float32)).cuda()
    P.ppca_split_f32(ctx, X, s.d); Xm = P.matrix(X, split=True)
    W = torch.zeros((w.m, s.d), device="cuda"); E = torch.zeros((w.k, s.d), device="cuda")
    th = P.ppca_prime_power(ctx, Xm, w.m, 6, w.init_seed, W, theta_hist=True); show(f"{name} values ")
    r = P.ppca_refine(ctx, Xm, W, w.m, w.k, E); show(f"{name} vectors")
    torch.cuda.synchronize()
    res[f"th_hist_{name}"] = th
    res[f"th_refine_{name}"] = np.asarray(r[0] if isinstance(r, tuple) else r, dtype=np.float64)
    res[f"E_{name}"] = E.cpu().numpy().astype(np.float64)
np.savez(f"/tmp/ritz_opt_{opt}.npz", **res)
