import numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_2109_03709_b200 as P
from tests import gpu_util as U
ctx = P.ppca_ctx_create(0, torch.cuda.current_stream())
rng = np.random.default_rng(6)
for n, d in [(301, 40), (64, 8), (300, 64)]:
    X = rng.standard_normal((n, d)).astype(np.float32)
    Xm = P.matrix(U.upload(X, "f32"))
    G = torch.zeros((d, d), dtype=torch.float64, device="cuda")
    P.ppca_gram(ctx, Xm, G)
    ref = X.astype(np.float64).T @ X.astype(np.float64)
    g = G.cpu().numpy()
    print(n, d, np.abs(g - ref).max(), g[:2, :4], ref[:2, :4])
