"""Thin Python binding of libppca.so (include/ppca.h) — argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; torch is used here only to
own device memory and streams (tensors are passed by pointer).  Functions keep the C names.
The binding fails loudly if the CUDA library is missing: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libppca.so")

PPCA_F32, PPCA_BF16, PPCA_F32_SPLIT = 0, 1, 2
PPCA_LAYOUT_CONTIGUOUS, PPCA_LAYOUT_INTERLEAVED = 0, 1
PPCA_PLANTED_QR, PPCA_PLANTED_HOUSEHOLDER, PPCA_IMAGE_FACTOR = 0, 1, 2
PPCA_SPECTRUM_EXP, PPCA_SPECTRUM_POWER = 0, 1
PPCA_UNIQUE_ID_BYTES = 128
PPCA_MAX_M = 128

STATUS = {0: "PPCA_OK", 1: "PPCA_ERR_INVALID_ARG", 2: "PPCA_ERR_DIM_MISMATCH", 3: "PPCA_ERR_TOO_MANY_COMPONENTS",
          4: "PPCA_ERR_NONFINITE", 5: "PPCA_ERR_DEGENERATE", 6: "PPCA_ERR_SUBSPACE_COLLAPSE",
          7: "PPCA_ERR_NO_CONVERGENCE", 8: "PPCA_ERR_CUDA", 9: "PPCA_ERR_NCCL", 10: "PPCA_ERR_UNSUPPORTED"}

# every symbol include/ppca.h declares (tests check the library exports all of them)
EXPORTS = ["ppca_status_string", "ppca_abi_version", "ppca_get_unique_id", "ppca_ctx_create", "ppca_ctx_destroy",
           "ppca_last_error", "ppca_launch_count", "ppca_generate", "ppca_prime_power", "ppca_prime_oja",
           "ppca_prime_eigengame", "ppca_refine", "ppca_eval", "ppca_captured_variance", "ppca_gram",
           "ppca_philox_words", "ppca_set_pass_impl", "ppca_set_timing", "ppca_get_pass_time",
           "ppca_last_pass_impl", "ppca_last_power_kernel", "ppca_split_f32", "ppca_upload_rows", "ppca_get_kernel_time", "ppca_refine_sampled",
           "ppca_check_prop3", "ppca_collective_count", "ppca_experiments_enabled", "ppca_ritz_residuals", "ppca_refine_ex",
           "ppca_check_theorem1", "ppca_set_orth_split"]


class PPCAError(RuntimeError):
    def __init__(self, status: int, msg: str):
        self.status = status
        self.name = STATUS.get(status, str(status))
        super().__init__(f"{self.name}: {msg}")


class ppca_matrix(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("dtype", ctypes.c_int), ("n_local", ctypes.c_int64),
                ("n_global", ctypes.c_int64), ("d", ctypes.c_int64), ("ld", ctypes.c_int64),
                ("layout", ctypes.c_int), ("block_rows", ctypes.c_int64)]


class ppca_gen_spec(ctypes.Structure):
    _fields_ = [("family", ctypes.c_int), ("spectrum", ctypes.c_int), ("a", ctypes.c_double),
                ("noise", ctypes.c_double), ("relu", ctypes.c_int32), ("house_r", ctypes.c_int32),
                ("rank", ctypes.c_int32), ("dtype", ctypes.c_int), ("n_global", ctypes.c_int64),
                ("d", ctypes.c_int64), ("seed", ctypes.c_uint64), ("layout", ctypes.c_int),
                ("block_rows", ctypes.c_int64)]


_lib = None


def load(path: str = LIB_PATH):
    """Load libppca.so (raises if it has not been built — there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"libppca.so not built at {path}: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    P, I64, I, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
    sig = {
        "ppca_status_string": (ctypes.c_char_p, [I]),
        "ppca_abi_version": (I, []),
        "ppca_get_unique_id": (I, [P]),
        "ppca_ctx_create": (I, [I, P, P, I, I, ctypes.POINTER(P)]),
        "ppca_ctx_destroy": (I, [P]),
        "ppca_last_error": (I, [P, ctypes.c_char_p, ctypes.c_size_t]),
        "ppca_launch_count": (I64, [P]),
        "ppca_generate": (I, [P, ctypes.POINTER(ppca_gen_spec), P, I64, ctypes.POINTER(I64), P]),
        "ppca_prime_power": (I, [P, ctypes.POINTER(ppca_matrix), I, I, D, ctypes.c_uint64, P, P, ctypes.POINTER(I)]),
        "ppca_collective_count": (I64, [P]),
        "ppca_set_orth_split": (I, [P, I]),
        "ppca_ritz_residuals": (I, [P, ctypes.POINTER(ppca_matrix), P, I, P, P, P]),
        "ppca_check_theorem1": (I, [P, ctypes.POINTER(ppca_matrix), P, I, I, P, D, ctypes.POINTER(I), P, P,
                                    ctypes.POINTER(I)]),
        "ppca_refine_ex": (I, [P, ctypes.POINTER(ppca_matrix), P, I, I, ctypes.c_uint, P, P, ctypes.POINTER(I)]),
        "ppca_experiments_enabled": (I, []),
        "ppca_prime_oja": (I, [P, ctypes.POINTER(ppca_matrix), I, I, D, D, I64, ctypes.c_uint64, P, P,
                               ctypes.POINTER(I64)]),
        "ppca_prime_eigengame": (I, [P, ctypes.POINTER(ppca_matrix), I, I, D, D, I64, ctypes.c_uint64, P, P,
                                     ctypes.POINTER(I64)]),
        "ppca_refine": (I, [P, ctypes.POINTER(ppca_matrix), P, I, I, P, P, ctypes.POINTER(I)]),
        "ppca_eval": (I, [P, P, P, I, I64, P, I, P, P]),
        "ppca_captured_variance": (I, [P, ctypes.POINTER(ppca_matrix), P, I, P]),
        "ppca_gram": (I, [P, ctypes.POINTER(ppca_matrix), P]),
        "ppca_philox_words": (I, [P, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64, I64, P]),
        "ppca_set_pass_impl": (I, [P, I]),
        "ppca_set_timing": (I, [P, I]),
        "ppca_last_pass_impl": (I, [P]),
        "ppca_last_power_kernel": (I, [P]),
        "ppca_upload_rows": (I, [P, P, I64, I64, ctypes.POINTER(ppca_matrix), I64]),
        "ppca_get_pass_time": (I, [P, ctypes.POINTER(D), ctypes.POINTER(I64)]),
        "ppca_split_f32": (I, [P, P, I64, I64, I64]),
        "ppca_refine_sampled": (I, [P, ctypes.POINTER(ppca_matrix), P, I, I, D, ctypes.c_uint64, P, P,
                                    ctypes.POINTER(I), ctypes.POINTER(I64)]),
        "ppca_get_kernel_time": (I, [P, I, ctypes.POINTER(D), ctypes.POINTER(I64)]),
        "ppca_check_prop3": (I, [P, ctypes.POINTER(ppca_matrix), P, I, P, I, D, P, P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


# ----------------------------------------------------------------------------- helpers
def _ptr(t) -> int:
    if t is None:
        return 0
    if t.dim() != 2 or not t.is_contiguous():
        raise ValueError("vector-set tensors must be contiguous 2-D [rows][d]")
    return int(t.data_ptr())


def _ptr1(t) -> int:
    if not t.is_contiguous():
        raise ValueError("output tensor must be contiguous")
    return int(t.data_ptr())


def _np_ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _check(ctx, status: int, what: str):
    if status != 0:
        msg = ""
        if ctx:
            buf = ctypes.create_string_buffer(512)
            _lib.ppca_last_error(ctx, buf, 512)
            msg = buf.value.decode(errors="replace")
        raise PPCAError(status, f"{what}: {msg}")


def matrix(X, n_global: int | None = None, layout: int = PPCA_LAYOUT_CONTIGUOUS, block_rows: int = 0,
           d: int | None = None, split: bool = False) -> ppca_matrix:
    """ppca_matrix for a 2-D CUDA tensor X [n_local][ld] (row-major; columns ≥ d are padding).
    split=True: a float32-sized tensor whose rows hold the PPCA_F32_SPLIT layout (ppca_split_f32)."""
    import torch
    if X.dim() != 2 or X.stride(1) != 1:
        raise ValueError("X must be a row-major 2-D tensor")
    if X.dtype == torch.float32:
        dt = PPCA_F32_SPLIT if split else PPCA_F32
    elif X.dtype == torch.bfloat16:
        dt = PPCA_BF16
    else:
        raise ValueError(f"unsupported dtype {X.dtype}")
    n_local = X.shape[0]
    mat = ppca_matrix(int(X.data_ptr()), dt, n_local, n_global if n_global is not None else n_local,
                      d if d is not None else X.shape[1], X.stride(0) if n_local > 0 else max(X.shape[1], 4),
                      layout, block_rows)
    mat._tensor = X          # keep the device buffer alive as long as the descriptor
    return mat


def gen_spec(spec, layout: int = PPCA_LAYOUT_CONTIGUOUS, block_rows: int = 0, split: bool = False) -> ppca_gen_spec:
    """ppca_gen_spec from an inputs.generate.GenSpec-like object (split=True: fp32 data written in the
    PPCA_F32_SPLIT layout)."""
    fam = {"planted_qr": PPCA_PLANTED_QR, "planted_householder": PPCA_PLANTED_HOUSEHOLDER,
           "image_factor": PPCA_IMAGE_FACTOR}[spec.family]
    return ppca_gen_spec(fam, PPCA_SPECTRUM_EXP if spec.spectrum == "exp" else PPCA_SPECTRUM_POWER, spec.a,
                         spec.noise, int(spec.relu), spec.house_r, spec.rank,
                         (PPCA_F32_SPLIT if split else PPCA_F32) if spec.dtype == "f32" else PPCA_BF16, spec.n, spec.d,
                         spec.seed, layout, block_rows)


# ----------------------------------------------------------------------------- multi-GPU plumbing
def contiguous_shard(n: int, rank: int, world: int) -> tuple[int, int]:
    """(first row, rows) of rank's CONTIGUOUS shard: rows [⌈n/G⌉·g, min(n, ⌈n/G⌉·(g+1))) (ppca.h)."""
    per = -(-n // world)
    r0 = min(n, per * rank)
    return r0, max(0, min(n, per * (rank + 1)) - r0)


def broadcast_unique_id(uid: bytes | None, group=None) -> bytes:
    """Rank 0's NCCL unique id (PPCA_UNIQUE_ID_BYTES bytes) delivered to every rank through the
    active torch.distributed process group (device tensor for nccl, host tensor for gloo)."""
    import torch
    import torch.distributed as dist
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.zeros(PPCA_UNIQUE_ID_BYTES, dtype=torch.uint8, device=dev)
    if dist.get_rank(group) == 0:
        if uid is None or len(uid) != PPCA_UNIQUE_ID_BYTES:
            raise ValueError("rank 0 must provide a PPCA_UNIQUE_ID_BYTES unique id")
        t.copy_(torch.frombuffer(bytearray(uid), dtype=torch.uint8))
    dist.broadcast(t, 0, group=group)
    return bytes(t.cpu().numpy().tobytes())


def ppca_ctx_create_distributed(local_rank: int, stream=None):
    """Collective: one context per rank of the active torch.distributed group (NCCL comm of the
    library bootstrapped from rank 0's unique id); world == 1 creates a plain context."""
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return ppca_ctx_create(local_rank, stream)
    rank, world = dist.get_rank(), dist.get_world_size()
    uid = broadcast_unique_id(ppca_get_unique_id() if rank == 0 else None)
    return ppca_ctx_create(local_rank, stream, uid, rank, world)


# ----------------------------------------------------------------------------- ABI (same names)
def ppca_status_string(s: int) -> str:
    return load().ppca_status_string(s).decode()


def ppca_abi_version() -> int:
    return load().ppca_abi_version()


def ppca_get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(PPCA_UNIQUE_ID_BYTES)
    _check(None, load().ppca_get_unique_id(buf), "ppca_get_unique_id")
    return buf.raw


def ppca_ctx_create(device: int = 0, stream=None, uid: bytes | None = None, rank: int = 0, world: int = 1):
    lib = load()
    h = ctypes.c_void_p()
    sp = ctypes.c_void_p(stream.cuda_stream if stream is not None else 0)
    ub = ctypes.create_string_buffer(uid, PPCA_UNIQUE_ID_BYTES) if uid is not None else None
    _check(None, lib.ppca_ctx_create(device, sp, ub, rank, world, ctypes.byref(h)), "ppca_ctx_create")
    return h


def ppca_ctx_destroy(ctx) -> None:
    _check(None, load().ppca_ctx_destroy(ctx), "ppca_ctx_destroy")


def ppca_launch_count(ctx) -> int:
    return int(load().ppca_launch_count(ctx))


def ppca_set_orth_split(ctx, split: int) -> None:
    _check(ctx, load().ppca_set_orth_split(ctx, split), "ppca_set_orth_split")


def ppca_collective_count(ctx) -> int:
    return int(load().ppca_collective_count(ctx))


def ppca_experiments_enabled() -> bool:
    return bool(load().ppca_experiments_enabled())


def ppca_ctx_create_one_rank_comm(device: int = 0, stream=None):
    """A world-1 context WITH a one-rank NCCL communicator: every all-reduce call site of the path runs
    (tests of the multi-GPU data plane on one GPU)."""
    return ppca_ctx_create(device, stream, ppca_get_unique_id(), 0, 1)


def ppca_set_pass_impl(ctx, impl: int) -> None:
    _check(ctx, load().ppca_set_pass_impl(ctx, impl), "ppca_set_pass_impl")


def ppca_last_pass_impl(ctx) -> int:
    return int(load().ppca_last_pass_impl(ctx))


def ppca_last_power_kernel(ctx) -> int:
    return int(load().ppca_last_power_kernel(ctx))


def ppca_set_timing(ctx, enable: bool) -> None:
    _check(ctx, load().ppca_set_timing(ctx, int(enable)), "ppca_set_timing")


def ppca_get_pass_time(ctx) -> tuple[float, int]:
    ms, n = ctypes.c_double(), ctypes.c_int64()
    _check(ctx, load().ppca_get_pass_time(ctx, ctypes.byref(ms), ctypes.byref(n)), "ppca_get_pass_time")
    return ms.value, n.value


def ppca_get_kernel_time(ctx, which: int) -> tuple[float, int]:
    """(summed ms, launches) of tensor-core kernel A (which=0) or B (which=1) since the last call."""
    ms, n = ctypes.c_double(), ctypes.c_int64()
    _check(ctx, load().ppca_get_kernel_time(ctx, which, ctypes.byref(ms), ctypes.byref(n)), "ppca_get_kernel_time")
    return ms.value, n.value


def ppca_generate(ctx, spec: ppca_gen_spec, X) -> tuple[int, np.ndarray]:
    """Fill the CUDA tensor X (this rank's shard, [n_local][ld]); returns (n_local, column mean)."""
    n_local = ctypes.c_int64()
    mean = np.zeros(spec.d, dtype=np.float64)
    _check(ctx, load().ppca_generate(ctx, ctypes.byref(spec), int(X.data_ptr()), X.stride(0), ctypes.byref(n_local),
                                     _np_ptr(mean)), "ppca_generate")
    return n_local.value, mean


def ppca_split_f32(ctx, X, d: int | None = None) -> None:
    """Convert the float32 CUDA tensor X [n_local][ld] in place to the PPCA_F32_SPLIT layout."""
    if X.dim() != 2 or X.stride(1) != 1:
        raise ValueError("X must be a row-major 2-D tensor")
    _check(ctx, load().ppca_split_f32(ctx, int(X.data_ptr()), X.shape[0], d if d is not None else X.shape[1],
                                      X.stride(0)), "ppca_split_f32")


def ppca_upload_rows(ctx, host, X: ppca_matrix, r0: int = 0) -> None:
    """Copy the rows of the host tensor `host` (row-major 2-D, CPU, fp32 for an fp32 / split X, bf16 for a bf16 X;
    pinned for an asynchronous copy) into the device shard X at local row r0 (split in place for PPCA_F32_SPLIT)."""
    if host.dim() != 2 or host.stride(1) != 1 or host.is_cuda:
        raise ValueError("host must be a row-major 2-D CPU tensor")
    _check(ctx, load().ppca_upload_rows(ctx, int(host.data_ptr()), host.shape[0], host.stride(0), ctypes.byref(X), r0),
           "ppca_upload_rows")


def ppca_prime_power_ex(ctx, X: ppca_matrix, m: int, iters: int, init_seed: int, W, theta_hist: bool = False,
                        eps: float = 0.0):
    """Block power priming with the paper's stop rule (eps > 0, P L61-62): (θ history rows run | None,
    iterations run)."""
    th = np.zeros((max(iters, 1), m), dtype=np.float64) if theta_hist else None
    done = ctypes.c_int()
    _check(ctx, load().ppca_prime_power(ctx, ctypes.byref(X), m, iters, float(eps), init_seed, _ptr(W),
                                        _np_ptr(th) if th is not None else None, ctypes.byref(done)),
           "ppca_prime_power")
    return (th[:done.value] if th is not None else None), done.value


def ppca_prime_power(ctx, X: ppca_matrix, m: int, iters: int, init_seed: int, W, theta_hist: bool = False):
    return ppca_prime_power_ex(ctx, X, m, iters, init_seed, W, theta_hist)[0]


def ppca_prime_oja(ctx, X: ppca_matrix, m: int, batch: int, alpha: float, momentum: float, steps: int,
                   init_seed: int, W, velocity, step: int = 0) -> int:
    s = ctypes.c_int64(step)
    _check(ctx, load().ppca_prime_oja(ctx, ctypes.byref(X), m, batch, alpha, momentum, steps, init_seed, _ptr(W),
                                      _ptr(velocity), ctypes.byref(s)), "ppca_prime_oja")
    return s.value


def ppca_prime_eigengame(ctx, X: ppca_matrix, m: int, batch: int, alpha: float, momentum: float, steps: int,
                         init_seed: int, V, velocity, step: int = 0) -> int:
    s = ctypes.c_int64(step)
    _check(ctx, load().ppca_prime_eigengame(ctx, ctypes.byref(X), m, batch, alpha, momentum, steps, init_seed,
                                            _ptr(V), _ptr(velocity), ctypes.byref(s)), "ppca_prime_eigengame")
    return s.value


def ppca_refine(ctx, X: ppca_matrix, V, m: int, k: int, E) -> tuple[np.ndarray, int]:
    theta = np.zeros(k, dtype=np.float64)
    dim = ctypes.c_int()
    _check(ctx, load().ppca_refine(ctx, ctypes.byref(X), _ptr(V), m, k, _ptr(E), _np_ptr(theta),
                                   ctypes.byref(dim)), "ppca_refine")
    return theta, dim.value


PPCA_REFINE_ORTHONORMAL = 1


def ppca_refine_ex(ctx, X: ppca_matrix, V, m: int, k: int, E, flags: int = 0) -> tuple[np.ndarray, int]:
    theta = np.zeros(k, dtype=np.float64)
    dim = ctypes.c_int()
    _check(ctx, load().ppca_refine_ex(ctx, ctypes.byref(X), _ptr(V), m, k, flags, _ptr(E), _np_ptr(theta),
                                      ctypes.byref(dim)), "ppca_refine_ex")
    return theta, dim.value


def ppca_refine_sampled(ctx, X: ppca_matrix, V, m: int, k: int, E, fraction: float,
                        sample_seed: int) -> tuple[np.ndarray, int, int]:
    """Row-subsampled refine: (θ rescaled to the full data, subspace dim, rows used)."""
    theta = np.zeros(k, dtype=np.float64)
    dim = ctypes.c_int()
    used = ctypes.c_int64()
    _check(ctx, load().ppca_refine_sampled(ctx, ctypes.byref(X), _ptr(V), m, k, fraction, sample_seed, _ptr(E),
                                           _np_ptr(theta), ctypes.byref(dim), ctypes.byref(used)),
           "ppca_refine_sampled")
    return theta, dim.value, used.value


def ppca_check_prop3(ctx, X: ppca_matrix, V, m: int, T, upto: int, tol: float = 1e-8) -> tuple[list, np.ndarray]:
    """Proposition 3 conditions 1 … upto (P L293–302): (flags, angles); flags[i] = conditions 1 … i hold."""
    ang = np.zeros(upto, dtype=np.float64)
    fl = np.zeros(upto, dtype=np.int32)
    _check(ctx, load().ppca_check_prop3(ctx, ctypes.byref(X), _ptr(V), m, _ptr(T), upto, tol, _np_ptr(ang),
                                        _np_ptr(fl)), "ppca_check_prop3")
    return [bool(f) for f in fl], ang


def ppca_check_theorem1(ctx, X: ppca_matrix, V, m: int, k: int, T, tol: float = 1e-8):
    """Theorem 1 online assertion (P L308-312): (upto, priming angles, pPCA angles, holds)."""
    upto, holds = ctypes.c_int(), ctypes.c_int()
    ap = np.zeros(k, dtype=np.float64)
    aq = np.zeros(k, dtype=np.float64)
    _check(ctx, load().ppca_check_theorem1(ctx, ctypes.byref(X), _ptr(V), m, k, _ptr(T), tol, ctypes.byref(upto),
                                           _np_ptr(ap), _np_ptr(aq), ctypes.byref(holds)), "ppca_check_theorem1")
    return upto.value, ap, aq, bool(holds.value)


def ppca_eval(ctx, E, T, k: int, d: int, thresholds) -> tuple[np.ndarray, np.ndarray]:
    thr = np.ascontiguousarray(thresholds, dtype=np.float64)
    ang = np.zeros(k, dtype=np.float64)
    lc = np.zeros(len(thr), dtype=np.int32)
    _check(ctx, load().ppca_eval(ctx, _ptr(E), _ptr(T), k, d, _np_ptr(thr), len(thr), _np_ptr(ang), _np_ptr(lc)),
           "ppca_eval")
    return ang, lc


def ppca_ritz_residuals(ctx, X: ppca_matrix, E, k: int, theta, gram: bool = False):
    """‖XᵀX e_i − θ_i e_i‖ for the rows of E (certification support, reading R29); gram=True also returns the
    k×k Gram of the residual rows (‖R‖₂² = its largest eigenvalue)."""
    th = np.ascontiguousarray(theta[:k], dtype=np.float64)
    out = np.zeros(k, dtype=np.float64)
    rg = np.zeros((k, k), dtype=np.float64) if gram else None
    _check(ctx, load().ppca_ritz_residuals(ctx, ctypes.byref(X), _ptr(E), k, _np_ptr(th), _np_ptr(out),
                                           _np_ptr(rg) if gram else None), "ppca_ritz_residuals")
    return (out, rg) if gram else out


def ppca_captured_variance(ctx, X: ppca_matrix, V, m: int) -> np.ndarray:
    out = np.zeros(m, dtype=np.float64)
    _check(ctx, load().ppca_captured_variance(ctx, ctypes.byref(X), _ptr(V), m, _np_ptr(out)),
           "ppca_captured_variance")
    return out


def ppca_gram(ctx, X: ppca_matrix, G) -> None:
    _check(ctx, load().ppca_gram(ctx, ctypes.byref(X), _ptr(G)), "ppca_gram")


def ppca_philox_words(ctx, seed: int, stream: int, first: int, out) -> None:
    _check(ctx, load().ppca_philox_words(ctx, seed, stream, first, out.numel(), _ptr1(out)), "ppca_philox_words")
