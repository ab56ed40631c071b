"""ORACLE — plain, slow, fp64 CPU implementation of primed PCA (arXiv 2109.03709).

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import this module.
The product path (`paper_2109_03709_b200`, the C-ABI library `libppca.so`)
never imports, links or calls anything here, and this module shares no code
with it: the only thing both sides consume is the seeded input generator in
`inputs/`, which holds none of the method's arithmetic.

Everything is fp64 numpy with one operation per line in the paper's order.
Vector sets are stored as [m][d] arrays (row i = vector v_i), matching the ABI.
Citations: "P Lnn" = reference PAPER.md line nn, "S Lnn" = reference SPEC.md line nn,
readings R1..R* = DESIGN.md §Readings.

Pins (tests/test_oracle_*.py, `-m "not gpu"`): see DESIGN.md §Oracle pins.  The
minibatch trajectories (prime_oja / prime_eigengame) are pinned only through
fixed points, monotonicity, single-step hand values and the Nesterov unroll;
beyond that their multi-step trajectory is "parity unpinned".
"""
from __future__ import annotations

import math
import numpy as np


class OracleError(RuntimeError):
    pass


class SubspaceCollapse(OracleError):
    """S L332: fewer than k primed directions survive orthonormalisation."""


class Degenerate(OracleError):
    """S L243 (EigenGame denominator) / S L225 (zero vector)."""


class NonFinite(OracleError):
    """S L234: a priming update produced a non-finite weight."""


class NoConvergence(OracleError):
    """S L61: Jacobi exceeded its sweep budget."""


# =============================================================================
# linalg
# =============================================================================
def gram_schmidt(V: np.ndarray, drop_tol: float = 1e-10, drop: bool = True) -> np.ndarray:
    """Orthonormal basis of span(rows of V): modified Gram–Schmidt with one
    re-orthogonalisation pass; rows whose residual norm is < drop_tol are dropped
    (S L48–51).  Realises Alg. 1 step 2 "V ← span(v_1,…,v_{k+l})" (P L48) and the
    "orthogonalize after every training step" of the multi-component power method
    (P L63).  Surviving rows keep their order; with drop=False a collapse raises."""
    out = []
    for v in np.asarray(V, dtype=np.float64):
        w = v.copy()
        for _ in range(2):                       # MGS + one reorthogonalisation
            for b in out:
                w = w - (b @ w) * b
        nrm = math.sqrt(w @ w)
        if nrm < drop_tol:
            if drop:
                continue
            raise SubspaceCollapse("vector collapsed during Gram–Schmidt")
        out.append(w / nrm)
    return np.array(out).reshape(len(out), np.asarray(V).shape[1])


def sign_convention(E: np.ndarray) -> np.ndarray:
    """Each row's entry of largest |value| made positive, ties → lowest index (S L60, R15)."""
    E = np.array(E, dtype=np.float64, copy=True)
    for i in range(E.shape[0]):
        j = int(np.argmax(np.abs(E[i])))          # argmax returns the first maximal index
        if E[i, j] < 0:
            E[i] = -E[i]
    return E


def jacobi_eigh(A: np.ndarray, tol: float = 1e-12, max_sweeps: int = 100):
    """Cyclic Jacobi eigen-decomposition of a symmetric matrix (S L57–61): the exact
    "full-PCA" of Alg. 1 step 4 (P L50).  Row-cyclic ordering, classical 2×2 symmetric
    Schur rotation (Golub & Van Loan, Alg. 8.4.2/8.4.3).  Stops when
    off(A) < tol·‖diag A‖_F.  Returns (eigenvalues descending — ties by original
    index — , eigenvectors as ROWS with the sign convention)."""
    A = np.array(A, dtype=np.float64, copy=True)
    n = A.shape[0]
    Vm = np.eye(n)
    for sweep in range(max_sweeps + 1):
        off = math.sqrt(np.sum((A - np.diag(np.diag(A))) ** 2))
        dia = math.sqrt(np.sum(np.diag(A) ** 2))
        if off <= tol * dia or off == 0.0:
            break
        if sweep == max_sweeps:
            raise NoConvergence(f"Jacobi: off={off:.3e} after {max_sweeps} sweeps")
        for p in range(n - 1):
            for q in range(p + 1, n):
                apq = A[p, q]
                if apq == 0.0:
                    continue
                tau = (A[q, q] - A[p, p]) / (2.0 * apq)
                t = (1.0 if tau >= 0 else -1.0) / (abs(tau) + math.sqrt(1.0 + tau * tau))
                c = 1.0 / math.sqrt(1.0 + t * t)
                s = t * c
                # A ← Jᵀ A J with J the rotation in the (p, q) plane
                ap, aq = A[:, p].copy(), A[:, q].copy()
                A[:, p] = c * ap - s * aq
                A[:, q] = s * ap + c * aq
                ap, aq = A[p, :].copy(), A[q, :].copy()
                A[p, :] = c * ap - s * aq
                A[q, :] = s * ap + c * aq
                vp, vq = Vm[:, p].copy(), Vm[:, q].copy()
                Vm[:, p] = c * vp - s * vq
                Vm[:, q] = s * vp + c * vq
    vals = np.diag(A).copy()
    order = np.argsort(-vals, kind="stable")
    return vals[order], sign_convention(Vm[:, order].T)


def normalize_rows(W: np.ndarray) -> np.ndarray:
    """current_components (S L266–270): each vector scaled to unit norm."""
    W = np.asarray(W, dtype=np.float64)
    nrm = np.sqrt(np.sum(W * W, axis=1))
    if np.any(nrm < 1e-300):
        raise Degenerate("zero vector")
    return W / nrm[:, None]


# =============================================================================
# priming (P §2; S L194–298)
# =============================================================================
def init_vectors(raw_gaussians: np.ndarray) -> np.ndarray:
    """S L212–215: i.i.d. N(0,1) vectors (drawn by inputs.generate.init_gaussians) scaled
    to unit norm (P L61 "initialises a random vector x_0 of unit norm")."""
    return normalize_rows(raw_gaussians)


def nesterov_update(param, velocity, direction, alpha, mu):
    """SGD with Nesterov momentum, ascent form (P L326; S L257–260):
    velocity ← μ·velocity + direction;  param ← param + α·(direction + μ·velocity)."""
    velocity = mu * velocity + direction
    param = param + alpha * (direction + mu * velocity)
    return param, velocity


def power_step(X: np.ndarray, W: np.ndarray):
    """One simultaneous power iteration on M = XᵀX (P L61–63), streaming X instead of
    forming M (R8):  Y = X·Wᵀ,  Z = Yᵀ·X (rows are (M w_i)ᵀ),  S = YᵀY,  W' = GS(Z).
    S = W M Wᵀ is the pPCA projected Gram of the *input* iterate W (P L260–269)."""
    Y = X @ W.T
    Z = Y.T @ X
    S = Y.T @ Y
    W_new = gram_schmidt(Z, drop=False)
    return W_new, S


def column_moves(W_new: np.ndarray, W_old: np.ndarray) -> np.ndarray:
    """‖x_{i+1} − x_i‖ of the stop rule (P L61-62) for every column of the block, sign-aligned: a column is
    an eigen-direction estimate defined up to sign, so min(‖w' − w‖, ‖w' + w‖)."""
    return np.array([min(np.linalg.norm(W_new[j] - W_old[j]), np.linalg.norm(W_new[j] + W_old[j]))
                     for j in range(W_new.shape[0])])


def prime_power(X: np.ndarray, W0_raw: np.ndarray, iters: int, eps: float = 0.0):
    """Block power priming: W_0 = GS(normalised Gaussians), then at most `iters` power steps.  eps > 0: the
    power method "terminates when ‖x_i − x_{i+1}‖ < ε" (P L61-62), here once every column moved less than
    eps (column_moves).  Returns (W_final, [S_0 … S_{t-1}]) — one S per iteration run."""
    W = gram_schmidt(init_vectors(W0_raw), drop=False)
    S_hist = []
    for _ in range(iters):
        W_new, S = power_step(X, W)
        S_hist.append(S)
        moved = column_moves(W_new, W)
        W = W_new
        if eps > 0 and np.max(moved) < eps:
            break
    return W, S_hist


def oja_step(Xb: np.ndarray, W: np.ndarray, vel: np.ndarray, alpha: float, mu: float):
    """Generalised Oja / Sanger minibatch step (P L70–72:
    Δw_m = α y_m (x − Σ_{l≤m} y_l w_l)), summed over the rows of the batch (R8):
        Y = X_b Wᵀ;   G_m = Σ_r y_rm x_r − Σ_{l≤m} (Σ_r y_rm y_rl) w_l;
    followed by the Nesterov update (P L326).  Weights are not renormalised (S L233)."""
    Y = Xb @ W.T                               # y_rm = <w_m, x_r>
    YtY = Y.T @ Y
    m = W.shape[0]
    G = np.zeros_like(W)
    for mm in range(m):
        G[mm] = Y[:, mm] @ Xb                  # Σ_r y_rm x_r
        for ll in range(mm + 1):               # Σ_{l ≤ m}
            G[mm] -= YtY[mm, ll] * W[ll]
    W_new, vel_new = nesterov_update(W, vel, G, alpha, mu)
    if not np.all(np.isfinite(W_new)):
        raise NonFinite("Oja update diverged")
    return W_new, vel_new


def eigengame_utilities(M: np.ndarray, V: np.ndarray) -> np.ndarray:
    """EigenGame utilities, Eqs. (1)–(3) (P L76–88):
    U_j = v_jᵀMv_j − Σ_{i<j} (v_jᵀMv_i)² / (v_iᵀMv_i)."""
    m = V.shape[0]
    U = np.zeros(m)
    for j in range(m):
        U[j] = V[j] @ M @ V[j]
        for i in range(j):
            den = V[i] @ M @ V[i]
            if den <= 1e-12:
                raise Degenerate("EigenGame denominator")
            U[j] -= (V[j] @ M @ V[i]) ** 2 / den
    return U


def eigengame_step(Xb: np.ndarray, V: np.ndarray, vel: np.ndarray, alpha: float, mu: float):
    """α-EigenGame minibatch step (utilities P L76–88; update rule R11 / S L251):
    M_b = X_bᵀX_b (unnormalised, S L284);
    ∇_j = 2 M_b v_j − 2 Σ_{i<j} (v_jᵀM_b v_i)/(v_iᵀM_b v_i) · M_b v_i   (∂U_j/∂v_j, parents fixed);
    r_j = ∇_j − <∇_j, v_j> v_j   (projection onto the sphere's tangent space);
    Nesterov on r (P L326), then v_j ← v_j/‖v_j‖.  All players use the pre-step V."""
    Y = Xb @ V.T                               # y_rj = <v_j, x_r>
    MV = Y.T @ Xb                              # row j = (M_b v_j)ᵀ
    A = MV @ V.T                               # A_ij = (M_b v_i)·v_j = v_iᵀ M_b v_j
    amax = np.max(np.diag(A))
    m = V.shape[0]
    R = np.zeros_like(V)
    for j in range(m):
        g = 2.0 * MV[j]
        for i in range(j):
            if A[i, i] <= 1e-12 * amax:        # R12: relative threshold
                raise Degenerate("EigenGame denominator v_iᵀM v_i too small")
            g = g - 2.0 * (A[j, i] / A[i, i]) * MV[i]
        R[j] = g - (g @ V[j]) * V[j]
    V_new, vel_new = nesterov_update(V, vel, R, alpha, mu)
    if not np.all(np.isfinite(V_new)):
        raise NonFinite("EigenGame update diverged")
    return normalize_rows(V_new), vel_new


def minibatch_blocks(n: int, b: int):
    """Block schedule (R10): global step s uses rows [(s mod nb)·b, min(n, ·+b)); the last,
    partial block is kept.  Rows are i.i.d. by construction, so the fixed block order
    replaces SPEC's per-epoch reshuffle (S L125) and is identical for every GPU count."""
    nb = -(-n // b)
    return [(s * b, min(n, (s + 1) * b)) for s in range(nb)]


def prime_oja(X, W0_raw, batch, alpha, mu, steps, W=None, vel=None):
    """Generalised-Oja priming for `steps` minibatch steps (P L70–72, L326)."""
    W = init_vectors(W0_raw) if W is None else W
    vel = np.zeros_like(W) if vel is None else vel
    blocks = minibatch_blocks(X.shape[0], batch)
    for s in range(steps):
        r0, r1 = blocks[s % len(blocks)]
        W, vel = oja_step(X[r0:r1], W, vel, alpha, mu)
    return W, vel


def prime_eigengame(X, V0_raw, batch, alpha, mu, steps, V=None, vel=None):
    """α-EigenGame priming for `steps` minibatch steps (P L74–91, L326)."""
    V = init_vectors(V0_raw) if V is None else V
    vel = np.zeros_like(V) if vel is None else vel
    blocks = minibatch_blocks(X.shape[0], batch)
    for s in range(steps):
        r0, r1 = blocks[s % len(blocks)]
        V, vel = eigengame_step(X[r0:r1], V, vel, alpha, mu)
    return V, vel


# =============================================================================
# pPCA (Algorithm 1, P L41–54; S L300–366)
# =============================================================================
def projected_gram(X: np.ndarray, B: np.ndarray) -> np.ndarray:
    """Alg. 1 step 3 + the projected covariance (S L319–322): coordinates of the projected
    rows in the orthonormal basis B are Y = X·Bᵀ (π_S(x) is never formed, S L353);
    returns YᵀY (unnormalised; = X̃ᵀX̃ in basis B, P L260–269)."""
    Y = X @ B.T
    return Y.T @ Y


def ppca_refine(X: np.ndarray, V: np.ndarray, k: int):
    """pPCA_l (Alg. 1, P L47–51): B = orth(V) (drop < 1e-10), S = (XBᵀ)ᵀ(XBᵀ),
    (θ, U) = Jacobi(S), e_i = Σ_j U_ij b_j for i ≤ k, sign convention.
    Returns (E [k][d], θ[:k], θ all, subspace_dim)."""
    B = gram_schmidt(V, drop_tol=1e-10, drop=True)
    if B.shape[0] < k:
        raise SubspaceCollapse(f"only {B.shape[0]} of {k} directions survive")
    S = projected_gram(X, B)
    theta, U = jacobi_eigh(S)                  # U rows = eigenvectors (coordinates in B)
    E = U[:k] @ B                              # lift back to R^d
    E = sign_convention(E)
    return E, theta[:k], theta, B.shape[0]


SAMPLE_TILE = 128          # rows per sampling unit (R25)
STREAM_SAMPLE = 7          # Philox stream of the row-tile sample (R25)


def sampled_rows(n: int, fraction: float, seed: int) -> np.ndarray:
    """R25 (P L378 "we only project 10% of the data"): the row blocks [128t, 128t+128) ∩ [0, n) whose
    uniform U(seed, stream 7, key = 128t, the global index of the block's first row) is below `fraction`
    (the random numbers are inputs: inputs.philox)."""
    from inputs import philox as ph
    nt = -(-n // SAMPLE_TILE)
    u = ph.uniforms_at(seed, STREAM_SAMPLE, np.arange(nt, dtype=np.uint64) * SAMPLE_TILE)
    keep = np.nonzero(u < fraction)[0]
    if keep.size == 0:
        return np.zeros(0, dtype=np.int64)
    return np.concatenate([np.arange(t * SAMPLE_TILE, min(n, (t + 1) * SAMPLE_TILE)) for t in keep])


def ppca_refine_sampled(X: np.ndarray, V: np.ndarray, k: int, fraction: float, seed: int):
    """Row-subsampled pPCA (P L378): Alg. 1 with the projected covariance formed
    from a seeded fraction of the rows and rescaled by n / rows used, so θ estimate XᵀX's eigenvalues
    (the rescale leaves the eigenvectors unchanged).  Returns (E, θ[:k], rows used)."""
    rows = sampled_rows(X.shape[0], fraction, seed) if fraction < 1.0 else np.arange(X.shape[0])
    if rows.size == 0:
        raise OracleError("empty row sample")
    E, theta, _, _ = ppca_refine(X[rows], V, k)
    return E, theta * (X.shape[0] / rows.size), rows.size


class DegenerateProjection(OracleError):
    """S L343: some π_S(e_i) has norm < 1e-10 (relative to ‖e_i‖)."""


def check_prop3(X: np.ndarray, V: np.ndarray, T: np.ndarray, upto: int, tol: float = 1e-8):
    """Proposition 3 (P L293–302; S L337–345).  S = span V with orthonormal basis
    B = orth(V); C' = (XBᵀ)ᵀ(XBᵀ) is the projected covariance in B (P L260–269); y_i = B t_i are the
    coordinates of π_S(e_i) (t_i = the i-th true eigenvector, a row of T).  Condition i (1-based):
    π_S(e_i) maximises Var on the orthogonal complement (within S) of span(π_S(e_1), …, π_S(e_{i−1}))
    (P L296–300, reading R22's bullet end), tested as: the top eigenvector u_i of P_i C' P_i, with
    P_i = I − Q_iQ_iᵀ and Q_i an orthonormal basis of y_1 … y_{i−1}, is within angle `tol` of y_i.
    Returns (flags, angles): angles[i] = ∠(u_i, y_i) in [0, π/2] for every i ≤ upto; flags[i] is
    true iff conditions 1 … i all hold (S L343: "stops marking true at the first failure"; reading R28).
    A library eigensolver (numpy.linalg.eigh) serves as the eigen step."""
    X = np.asarray(X, dtype=np.float64)
    T = np.asarray(T, dtype=np.float64)
    if T.shape[0] < upto:
        raise OracleError("truth has fewer than `upto` vectors")
    B = gram_schmidt(V, drop_tol=1e-10, drop=True)
    C = projected_gram(X, B)                              # C' in basis B
    m = B.shape[0]
    flags, angs = [], []
    chain = True
    for i in range(upto):
        y = B @ T[i]                                      # π_S(e_i) in basis B
        if math.sqrt(y @ y) < 1e-10 * math.sqrt(T[i] @ T[i]):
            raise DegenerateProjection(f"|pi_S(e_{i + 1})| < 1e-10")
        Q = gram_schmidt(np.array([B @ T[j] for j in range(i)]).reshape(i, m), drop_tol=1e-10, drop=True)
        P = np.eye(m) - Q.T @ Q                           # projector onto the complement in S
        M = P @ C @ P
        w, U = np.linalg.eigh(M)
        u = U[:, int(np.argmax(w))]                       # the variance maximiser on the complement
        yh = y / math.sqrt(y @ y)
        c = abs(float(u @ yh))
        s = float(np.linalg.norm(u - (u @ yh) * yh))      # sine, accurate at tiny angles
        a = math.atan2(s, c)
        angs.append(a)
        chain = chain and a <= tol
        flags.append(chain)
    return flags, np.array(angs)


def theorem1_check(X: np.ndarray, V: np.ndarray, T: np.ndarray, k: int, tol: float = 1e-8):
    """Theorem 1 (P L308-312) as an online assertion: for the priming output V (m ≥ k
    vectors, e_i^PRIMING = v_i/‖v_i‖ for i ≤ k) and the true eigenvectors T, let `upto` be the length of the
    leading run of Proposition 3's conditions that hold (check_prop3 flags, P L293-302).  On that run the
    full-PCA step returns π_S(e_i)/‖π_S(e_i)‖ as its i-th vector (Prop. 1 / Prop. 3's proof, P L287-306) —
    the vector of S closest to e_i — so it cannot be farther from e_i than the priming's own v_i ∈ S:
        ∠(pPCA_i, e_i) ≤ ∠(v_i, e_i) + tol   for every i ≤ upto,
    hence LCES(pPCA) ≥ LCES(priming) on that run for every threshold V.  Returns (upto, angles of the priming
    vectors, angles of the pPCA vectors, holds)."""
    flags, _ = check_prop3(X, V, T, k, tol)
    upto = 0
    while upto < k and flags[upto]:
        upto += 1
    E, _, _, _ = ppca_refine(X, V, k)
    Vn = normalize_rows(np.asarray(V, dtype=np.float64)[:k])
    a_prim = angles(Vn, T[:k])
    a_ppca = angles(E, T[:k])
    holds = all(a_ppca[i] <= a_prim[i] + tol for i in range(upto))
    return upto, a_prim, a_ppca, holds


def ritz_values(S: np.ndarray) -> np.ndarray:
    """Ritz values of an orthonormal-basis Gram S (the pPCA eigenvalue estimates)."""
    return jacobi_eigh(S)[0]


# =============================================================================
# metrics (P §5.3; S L368–439)
# =============================================================================
PI_THRESHOLDS = [math.pi / 2 ** s for s in range(3, 11)]     # π/8 … π/1024 (P L413)


def angular_error(v: np.ndarray, e: np.ndarray) -> float:
    """arccos(min(1, |<v,e>|)) — sign-invariant angle (S L388)."""
    return math.acos(min(1.0, abs(float(np.dot(v, e)))))


def angles(E: np.ndarray, T: np.ndarray) -> np.ndarray:
    return np.array([angular_error(E[i], T[i]) for i in range(E.shape[0])])


def lces(angle_list, V: float) -> int:
    """Longest Correct Eigenvector Streak (P L412): number of consecutive indices from 1
    whose angle is strictly smaller than V."""
    s = 0
    for a in angle_list:
        if a < V:
            s += 1
        else:
            break
    return s


def captured_variance(X: np.ndarray, v: np.ndarray) -> float:
    """vᵀ(XᵀX)v computed as ‖Xv‖² (P L416 footnote; S L406)."""
    y = X @ v
    return float(y @ y)


def covariance(X: np.ndarray, normalize: bool = False) -> np.ndarray:
    """XᵀX (P L15), divided by n on request (P L198)."""
    C = X.T @ X
    return C / X.shape[0] if normalize else C


def truth(X: np.ndarray):
    """Ground truth (S L428): eigen-decomposition of the fp64 XᵀX of the stored data,
    descending, eigenvectors as rows with the sign convention.  Uses LAPACK
    (numpy.linalg.eigh) as a library primitive; pinned against jacobi_eigh."""
    C = covariance(X)
    w, U = np.linalg.eigh(C)
    order = np.argsort(-w, kind="stable")
    return w[order], sign_convention(U[:, order].T)


def subspace_error(E: np.ndarray, T: np.ndarray) -> float:
    """Subspace error of SURVEY §8(c) O8 / reading R20 (the C5 target): ‖(I − T_kᵀT_k) E_kᵀ‖₂ for
    row-orthonormal E_k, T_k [k][d] — the sine of the largest principal angle between span E and span T."""
    P = E.T - T.T @ (T @ E.T)
    return float(np.linalg.norm(P, 2))


def ritz_residuals(X: np.ndarray, E: np.ndarray, theta: np.ndarray) -> np.ndarray:
    """r_i = ‖XᵀX e_i − θ_i e_i‖₂ for the rows e_i of E, with XᵀX applied as Xᵀ(X e_i) (never formed):
    the quantity the Weyl / Davis–Kahan certificates of certified_top are built on (reading R29)."""
    X = np.asarray(X, dtype=np.float64)
    E = np.asarray(E, dtype=np.float64)
    ME = (X @ E.T).T @ X
    R = ME - np.asarray(theta, dtype=np.float64)[:, None] * E
    return np.sqrt(np.sum(R * R, axis=1))


def certified_top(X: np.ndarray, k: int, W0_raw: np.ndarray, max_iters: int = 500, rtol: float = 1e-9):
    """Residual-certified reference for the top-k eigenpairs of M = XᵀX when M is too large to form (SURVEY
    §8(c) O9; reading R29): block power iteration (P L61-63) on m = W0_raw.shape[0] > k vectors with a
    Rayleigh–Ritz step each iteration (Alg. 1, P L47-51), fp64, until every residual
    r_i = ‖M e_i − θ_i e_i‖ (i ≤ k) is ≤ rtol·θ_1 or max_iters.  One pass over X per iteration gives both the
    residuals of the current Ritz pairs and the next iterate (span M·E = span M·W).
    Bounds (returned, R29):
      weyl_i  = r_i                      — some eigenvalue of M lies in [θ_i − r_i, θ_i + r_i] (Weyl);
      gap_i   = min_{j≠i, j≤m} |θ_i − θ_j| − r_j, and θ_i − (θ_m + r_m) for the unresolved tail
                (assumes the m Ritz intervals hold the top-m eigenvalues: block power from a random start);
      angle_i = r_i / gap_i              — sin∠(e_i, true eigenvector i) (Davis–Kahan);
      subspace = ‖R_k‖₂ / δ, δ = θ_k − (θ_{k+1} + r_{k+1})  — sin of the largest principal angle between
                span E_k and the true top-k subspace (Davis–Kahan sinΘ).
    Returns a dict with theta, E (rows, sign convention), res, gap, angle_bound, subspace_bound, iters."""
    X = np.asarray(X, dtype=np.float64)
    m = W0_raw.shape[0]
    if not k < m:
        raise OracleError("certified_top needs m > k (the tail gap uses theta_{k+1})")
    W = gram_schmidt(init_vectors(W0_raw), drop=False)
    out = None
    for it in range(1, max_iters + 1):
        Y = X @ W.T                                        # one pass: Y = X Wᵀ …
        S = Y.T @ Y                                        # … S = W M Wᵀ
        w, U = np.linalg.eigh(S)                           # Rayleigh–Ritz (library eigensolver as a step)
        order = np.argsort(-w, kind="stable")
        theta, U = w[order], U[:, order].T                 # rows of U: eigenvectors of S
        E = U @ W                                          # Ritz vectors (orthonormal rows)
        ME = (Y @ U.T).T @ X                               # rows: (M e_i)ᵀ = (X e_i)ᵀ X
        R = ME - theta[:, None] * E                        # residual rows
        res = np.sqrt(np.sum(R * R, axis=1))
        out = (theta, E, R, res, it)
        if np.all(res[:k] <= rtol * theta[0]):
            break
        W = gram_schmidt(ME, drop=False)                   # next iterate: span(M E) = span(M W)
    theta, E, R, res, it = out
    gap = np.empty(k)
    for i in range(k):
        others = [abs(theta[i] - theta[j]) - res[j] for j in range(m) if j != i]
        gap[i] = min(min(others), theta[i] - (theta[m - 1] + res[m - 1]))
    delta = theta[k - 1] - (theta[k] + res[k])
    sub = float(np.linalg.norm(R[:k], 2)) / delta if delta > 0 else math.inf
    ang = np.where(gap > 0, res[:k] / np.where(gap > 0, gap, 1.0), math.inf)
    return {"theta": theta[:k], "E": sign_convention(E[:k]), "res": res[:k], "gap": gap,
            "angle_bound": ang, "subspace_bound": sub, "iters": it, "theta_all": theta, "res_all": res}


def relative_gaps(lam: np.ndarray) -> np.ndarray:
    """R19: two-sided relative eigengap g_i = min(λ_{i-1}−λ_i, λ_i−λ_{i+1})/λ_i (one-sided at the ends)."""
    lam = np.asarray(lam, dtype=np.float64)
    g = np.full(lam.size, np.inf)
    for i in range(lam.size):
        if i > 0:
            g[i] = min(g[i], lam[i - 1] - lam[i])
        if i + 1 < lam.size:
            g[i] = min(g[i], lam[i] - lam[i + 1])
        g[i] /= abs(lam[i]) if lam[i] != 0 else 1.0
    return g
