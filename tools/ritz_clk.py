"""Phase clocks of the Ritz (tridiagonal) kernel on a C3s refine and a power iterate (profiling)."""
import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2109_03709_b200 as P
from inputs import configs as C, generate as G
lib = P.load(os.environ["PPCA_EXP_LIB"]) if os.environ.get("PPCA_EXP_LIB") else P.load(); lib.ppca_debug_wait_counters.argtypes = [ctypes.c_void_p]
w = C.SMALL["C3s"]; s = w.spec
ctx = P.ppca_ctx_create(0, torch.cuda.current_stream())
X = torch.from_numpy(np.ascontiguousarray(G.dataset(s), dtype=np.float32)).cuda()
P.ppca_split_f32(ctx, X, s.d); Xm = P.matrix(X, split=True)
W = torch.zeros((w.m, s.d), device="cuda"); E = torch.zeros((w.k, s.d), device="cuda")
names = ["cholesky", "L^-1", "C=L^-1 S L^-T", "tridiag", "multisection", "inv-iteration", "back-transform"]
def show(tag):
    out = (ctypes.c_ulonglong * 16)(); lib.ppca_debug_wait_counters(out)
    c = [out[i] for i in range(8)]
    print(tag, "  ".join(f"{n} {(c[i+1]-c[i])/1.9e3:.1f}us" for i, n in enumerate(names) if c[i+1] > c[i]))
    h = [out[8 + i] for i in range(5)]
    print("   chol_inv:", "  ".join(f"{n} {(h[i+1]-h[i])/1.9e3:.1f}us" for i, n in
                                   enumerate(["stage", "cholesky", "L^-1", "store"])))
P.ppca_prime_power(ctx, Xm, w.m, 2, w.init_seed, W, theta_hist=True); show("values ")
P.ppca_refine(ctx, Xm, W, w.m, w.k, E); show("vectors")
