"""B200-native Iterative Hessian Sketch hot path (arXiv 1910.14166).

A thin ctypes binding over ``libihs.so`` (C ABI in ``include/ihs.h``; kernels in
``csrc/``, hand-written for sm_100a).  This module only marshals arguments:
torch tensors supply device memory and the current CUDA stream; every step of
the path (hash, sort, sketch, gradient, Gram, inner solve, error norms) runs in
the library's kernels.  There is no CPU fallback: if ``libihs.so`` is missing or
cannot run, every call raises.

Names follow the C ABI: ``ihs_hash``, ``ihs_sketch``, ``ihs_grad``,
``ihs_sketch_grad``, ``ihs_gram``, ``ihs_ols_update``, ``ihs_l1ball_update``,
``ihs_solve_ols``, ``ihs_solve_l1ball``, ``ihs_pred_err2``; NEXT-2 (penalised LASSO):
``ihs_lasso_update``, ``ihs_solve_lasso``.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
import threading

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libihs.so")
ABI_VERSION = 2

OK, ERR_INVALID_ARGUMENT, ERR_DIMENSION_MISMATCH, ERR_NOT_SPD, ERR_NOT_CONVERGED, ERR_CUDA, ERR_COMM, \
    ERR_OUT_OF_MEMORY, ERR_UNSUPPORTED = range(9)
COUNTSKETCH, SJLT = 0, 1
K_SORT, K_SKETCH, K_SJLT, K_CSR, K_GRAD, K_REDUCE, K_GRAM, K_CHOL, K_PG = range(9)
KERNEL_GROUPS = ("sort", "sketch", "sjlt", "csr", "grad", "reduce", "gram", "chol", "pg", "factor", "apply")
DENSE, CSR = 0, 1


class IhsError(RuntimeError):
    def __init__(self, status: int, what: str):
        msg = lib().ihs_status_string(status).decode() if _lib is not None else str(status)
        super().__init__(f"{what}: {msg} (status {status})")
        self.status = status


class SketchSpec(C.Structure):
    _fields_ = [("family", C.c_int32), ("s", C.c_int32), ("m", C.c_int64), ("seed", C.c_uint64)]


class Matrix(C.Structure):
    _fields_ = [("layout", C.c_int32), ("reserved", C.c_int32), ("n_rows", C.c_int64), ("n_cols", C.c_int64),
                ("row_offset", C.c_int64), ("values", C.c_void_p), ("row_ptr", C.c_void_p),
                ("col_idx", C.c_void_p), ("nnz", C.c_int64)]


class InnerCfg(C.Structure):
    _fields_ = [("max_inner", C.c_int32), ("power_iters", C.c_int32), ("inner_tol", C.c_double),
                ("lip_safety", C.c_double), ("warm_power_iters", C.c_int32), ("reserved", C.c_int32)]


class IterRecord(C.Structure):
    _fields_ = [("t_sketch_grad", C.c_double), ("t_comm", C.c_double), ("t_gram", C.c_double),
                ("t_solve", C.c_double), ("inner_iters", C.c_int32), ("status", C.c_int32)]


_EXPORTS = {
    "ihs_abi_version": (C.c_int, []),
    "ihs_status_string": (C.c_char_p, [C.c_int]),
    "ihs_ctx_create": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.c_void_p]),
    "ihs_ctx_destroy": (C.c_int, [C.c_void_p]),
    "ihs_ctx_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "ihs_ctx_synchronize": (C.c_int, [C.c_void_p]),
    "ihs_ctx_kernel_launches": (C.c_int64, [C.c_void_p]),
    "ihs_ctx_set_option": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int64]),
    "ihs_ctx_get_option": (C.c_int, [C.c_void_p, C.c_char_p, C.POINTER(C.c_int64)]),
    "ihs_ctx_set_profiling": (C.c_int, [C.c_void_p, C.c_int]),
    "ihs_ctx_profile": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_int64)]),
    "ihs_ctx_profile_reset": (C.c_int, [C.c_void_p]),
    "ihs_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "ihs_ctx_set_comm": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p]),
    "ihs_allreduce_sum": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64]),
    "ihs_allreduce_multimem": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int64,
                                         C.c_int64]),
    "ihs_hash": (C.c_int, [C.c_void_p, C.POINTER(SketchSpec), C.c_uint64, C.c_int64, C.c_int64, C.c_void_p,
                           C.c_void_p]),
    "ihs_sketch": (C.c_int, [C.c_void_p, C.POINTER(Matrix), C.POINTER(SketchSpec), C.c_uint64, C.c_void_p,
                             C.c_int]),
    "ihs_grad": (C.c_int, [C.c_void_p, C.POINTER(Matrix), C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]),
    "ihs_sketch_grad": (C.c_int, [C.c_void_p, C.POINTER(Matrix), C.POINTER(SketchSpec), C.c_uint64, C.c_void_p,
                                  C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]),
    "ihs_gram": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_double, C.c_void_p]),
    "ihs_small_step": (C.c_int, [C.c_void_p, C.POINTER(Matrix), C.c_void_p, C.POINTER(SketchSpec), C.c_uint64,
                                 C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "ihs_ols_update": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    "ihs_gram_ols_update": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_double, C.c_void_p,
                                      C.c_void_p, C.c_void_p, C.c_void_p]),
    "ihs_ols_factor": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_double, C.c_void_p]),
    "ihs_gram_lookahead": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_double, C.c_void_p]),
    "ihs_ols_apply": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    "ihs_ols_lookahead_step": (C.c_int, [C.c_void_p, C.POINTER(Matrix), C.POINTER(SketchSpec), C.c_uint64,
                                         C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                         C.c_void_p]),
    "ihs_l1ball_update": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_double,
                                    C.POINTER(InnerCfg), C.c_void_p, C.c_void_p]),
    "ihs_lasso_update": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_double,
                                   C.POINTER(InnerCfg), C.c_void_p, C.c_void_p]),
    "ihs_solve_lasso": (C.c_int, [C.c_void_p, C.POINTER(Matrix), C.c_void_p, C.c_double, C.POINTER(SketchSpec),
                                  C.c_int32, C.c_uint64, C.POINTER(InnerCfg), C.c_void_p, C.c_void_p, C.c_void_p,
                                  C.POINTER(IterRecord)]),
    "ihs_solve_ols": (C.c_int, [C.c_void_p, C.POINTER(Matrix), C.c_void_p, C.POINTER(SketchSpec), C.c_int32,
                                C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(IterRecord)]),
    "ihs_solve_l1ball": (C.c_int, [C.c_void_p, C.POINTER(Matrix), C.c_void_p, C.c_double, C.POINTER(SketchSpec),
                                   C.c_int32, C.c_uint64, C.POINTER(InnerCfg), C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.POINTER(IterRecord)]),
    "ihs_pred_err2": (C.c_int, [C.c_void_p, C.POINTER(Matrix), C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                                C.c_void_p]),
}

_lib = None
_lock = threading.Lock()


def lib() -> C.CDLL:
    """Load libihs.so.  Raises if it is absent: there is no fallback path."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                                   "(python paper_1910_14166_b200/build.py)")
            L = C.CDLL(LIB_PATH)
            for name, (res, args) in _EXPORTS.items():
                f = getattr(L, name)
                f.restype = res
                f.argtypes = args
            if L.ihs_abi_version() != ABI_VERSION:
                raise RuntimeError("libihs.so ABI version mismatch")
            _lib = L
    return _lib


def _check(st: int, what: str):
    if st != OK:
        raise IhsError(st, what)


def _p(t):
    if t is None:
        return None
    if isinstance(t, torch.Tensor):
        if not t.is_contiguous():
            raise ValueError("tensors passed to libihs must be contiguous")
        return C.c_void_p(t.data_ptr())
    return C.c_void_p(t)


@dataclasses.dataclass(frozen=True)
class Spec:
    """Sketch spec: CountSketch (s = 1) or SJLT with s nonzeros per column."""
    m: int
    s: int = 1
    seed: int = 0
    family: int | None = None

    def c(self) -> SketchSpec:
        fam = self.family if self.family is not None else (COUNTSKETCH if self.s == 1 else SJLT)
        return SketchSpec(fam, self.s, self.m, self.seed)


class Dense:
    """Dense row-major fp64 row block of A; row_offset = global index of row 0."""

    def __init__(self, A: torch.Tensor, row_offset: int = 0):
        if A.dtype != torch.float64 or A.dim() != 2:
            raise ValueError("A must be a 2-D float64 tensor")
        self.A = A.contiguous()
        self.row_offset = row_offset
        self.n, self.d = self.A.shape
        self.device = A.device

    def c(self) -> Matrix:
        return Matrix(DENSE, 0, self.n, self.d, self.row_offset, self.A.data_ptr(), None, None, 0)


class Csr:
    """CSR fp64 row block: row_ptr int64 (n+1, rebased to 0), col int32, val f64."""

    def __init__(self, row_ptr: torch.Tensor, col: torch.Tensor, val: torch.Tensor, d: int, row_offset: int = 0):
        if row_ptr.dtype != torch.int64 or col.dtype != torch.int32 or val.dtype != torch.float64:
            raise ValueError("CSR dtypes: row_ptr int64, col int32, val float64")
        self.row_ptr, self.col, self.val = row_ptr.contiguous(), col.contiguous(), val.contiguous()
        self.n, self.d, self.row_offset = row_ptr.numel() - 1, d, row_offset
        self.device = val.device

    def c(self) -> Matrix:
        return Matrix(CSR, 0, self.n, self.d, self.row_offset, self.val.data_ptr(), self.row_ptr.data_ptr(),
                      self.col.data_ptr(), self.val.numel())


def as_matrix(A):
    if isinstance(A, (Dense, Csr)):
        return A
    if isinstance(A, torch.Tensor):
        return Dense(A)
    if isinstance(A, tuple) and len(A) == 4:
        return Csr(*A)
    raise TypeError("A must be a Dense, Csr, 2-D tensor or (row_ptr, col, val, d)")


class Context:
    """One libihs context per (device, stream).  Binds to the current torch stream
    at each call (set_stream) so that tensors' stream semantics hold."""

    def __init__(self, device: int | torch.device | None = None):
        if isinstance(device, torch.device):
            device = device.index or 0
        self.device = torch.cuda.current_device() if device is None else int(device)
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            stream = torch.cuda.current_stream().cuda_stream
        _check(lib().ihs_ctx_create(C.byref(h), self.device, C.c_void_p(stream)), "ihs_ctx_create")
        self.h = h
        # Tensors read asynchronously on the library's factor stream (the SA of
        # ihs_ols_factor / ihs_gram_lookahead), kept alive until the call that
        # joins their result (keyed by the output's address) or synchronize():
        # torch's caching allocator does not see that stream.
        self._keep: dict[int, tuple] = {}

    def _hold(self, out: torch.Tensor, *tensors):
        self._keep[out.data_ptr()] = (out,) + tensors

    def _release(self, out) -> None:
        if out is not None:
            self._keep.pop(out.data_ptr() if isinstance(out, torch.Tensor) else int(out), None)

    def _bind(self):
        stream = torch.cuda.current_stream(self.device).cuda_stream
        _check(lib().ihs_ctx_set_stream(self.h, C.c_void_p(stream)), "ihs_ctx_set_stream")
        return self.h

    def synchronize(self):
        st = lib().ihs_ctx_synchronize(self._bind())
        self._keep.clear()
        _check(st, "ihs_ctx_synchronize")

    def status(self) -> int:
        """Synchronise and return (not raise) the pending device status."""
        st = lib().ihs_ctx_synchronize(self._bind())
        self._keep.clear()
        return st

    @property
    def kernel_launches(self) -> int:
        return int(lib().ihs_ctx_kernel_launches(self.h))

    def set_option(self, name: str, value: int):
        """Per-context option (ihs.h: lookahead, sjlt_onepass, ols_large, fuse_max_d, pg_warm, prefetch)."""
        _check(lib().ihs_ctx_set_option(self.h, name.encode(), int(value)), f"ihs_ctx_set_option({name})")

    def get_option(self, name: str) -> int:
        v = C.c_int64()
        _check(lib().ihs_ctx_get_option(self.h, name.encode(), C.byref(v)), f"ihs_ctx_get_option({name})")
        return v.value

    def set_profiling(self, enable: bool):
        _check(lib().ihs_ctx_set_profiling(self.h, int(enable)), "ihs_ctx_set_profiling")

    def profile(self, group: int):
        """(summed ms, launches) of one kernel group since the last reset."""
        ms, k = C.c_double(), C.c_int64()
        _check(lib().ihs_ctx_profile(self._bind(), group, C.byref(ms), C.byref(k)), "ihs_ctx_profile")
        return ms.value, k.value

    def profile_reset(self):
        _check(lib().ihs_ctx_profile_reset(self._bind()), "ihs_ctx_profile_reset")

    def set_comm(self, rank: int, world: int, unique_id: bytes | None):
        buf = None if unique_id is None else C.create_string_buffer(unique_id, 128)
        _check(lib().ihs_ctx_set_comm(self.h, rank, world, buf), "ihs_ctx_set_comm")

    def close(self):
        if getattr(self, "h", None):
            lib().ihs_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().ihs_nccl_unique_id(buf), "ihs_nccl_unique_id")
    return buf.raw


_default_ctx: dict[int, Context] = {}


def default_context(device=None) -> Context:
    dev = torch.cuda.current_device() if device is None else (device.index if isinstance(device, torch.device)
                                                               else int(device))
    if dev not in _default_ctx:
        _default_ctx[dev] = Context(dev)
    return _default_ctx[dev]


def _f64(n, device):
    return torch.empty(n, dtype=torch.float64, device=device)


# ------------------------------------------------------------------ a1
def ihs_allreduce_sum(buf: torch.Tensor, ctx: Context | None = None) -> torch.Tensor:
    """In-place sum of a float64 device tensor across the context's communicator (a3)."""
    ctx = ctx or default_context(buf.device)
    assert buf.dtype == torch.float64 and buf.is_cuda and buf.is_contiguous()
    _check(lib().ihs_allreduce_sum(ctx._bind(), _p(buf), buf.numel()), "ihs_allreduce_sum")
    return buf


def ihs_allreduce_multimem(mc_ptr: int, pads: torch.Tensor, rank: int, world: int, count: int, pad_slots: int,
                           ctx: Context | None = None) -> None:
    """a3 over NVLS: in-place sum of `count` doubles of a symmetric buffer whose
    multicast address is mc_ptr; pads = int64 device tensor of the ranks'
    signal-pad pointers (ihs.h)."""
    ctx = ctx or default_context(pads.device)
    _check(lib().ihs_allreduce_multimem(ctx._bind(), C.c_void_p(mc_ptr), _p(pads), rank, world, count, pad_slots),
           "ihs_allreduce_multimem")


def ihs_hash(spec: Spec, it: int, row_begin: int, count: int, ctx: Context | None = None, device=None):
    ctx = ctx or default_context(device)
    dev = torch.device("cuda", ctx.device)
    bucket = torch.empty(count * spec.s, dtype=torch.int32, device=dev)
    sign = torch.empty(count * spec.s, dtype=torch.int8, device=dev)
    sp = spec.c()
    _check(lib().ihs_hash(ctx._bind(), C.byref(sp), it, row_begin, count, _p(bucket), _p(sign)), "ihs_hash")
    return bucket.view(count, spec.s), sign.view(count, spec.s)


# ------------------------------------------------------------------ a2 / a5
def ihs_sketch(A, spec: Spec, it: int, out: torch.Tensor | None = None, ctx: Context | None = None,
               reduce: bool = False):
    """S^it A (m x d); reduce=True sums it over the context's communicator (ihs.h)."""
    A = as_matrix(A)
    ctx = ctx or default_context(A.device)
    SA = out if out is not None else _f64((spec.m, A.d), A.device)
    mc, sp = A.c(), spec.c()
    _check(lib().ihs_sketch(ctx._bind(), C.byref(mc), C.byref(sp), it, _p(SA), int(reduce)), "ihs_sketch")
    return SA


def ihs_grad(A, b: torch.Tensor, x: torch.Tensor, out: torch.Tensor | None = None, ctx: Context | None = None,
             reduce: bool = False):
    """A^T (b - A x); reduce=True sums it over the context's communicator."""
    A = as_matrix(A)
    ctx = ctx or default_context(A.device)
    g = out if out is not None else _f64(A.d, A.device)
    mc = A.c()
    _check(lib().ihs_grad(ctx._bind(), C.byref(mc), _p(b), _p(x), _p(g), int(reduce)), "ihs_grad")
    return g


def ihs_sketch_grad(A, spec: Spec, it: int, b, x, SA=None, g=None, ctx: Context | None = None,
                    reduce: bool = False):
    """Packed [SA | g] when SA/g are None: returns (pack, SA view, g view)."""
    A = as_matrix(A)
    ctx = ctx or default_context(A.device)
    pack = None
    if SA is None or g is None:
        pack = _f64(spec.m * A.d + A.d, A.device)
        SA = pack[: spec.m * A.d].view(spec.m, A.d)
        g = pack[spec.m * A.d:]
    mc, sp = A.c(), spec.c()
    _check(lib().ihs_sketch_grad(ctx._bind(), C.byref(mc), C.byref(sp), it, _p(b), _p(x), _p(SA), _p(g),
                                 int(reduce)), "ihs_sketch_grad")
    return pack, SA, g


# ------------------------------------------------------------------ a4
def ihs_gram(SA: torch.Tensor, scale: float = 1.0, out=None, ctx: Context | None = None):
    ctx = ctx or default_context(SA.device)
    m, d = SA.shape
    H = out if out is not None else _f64((d, d), SA.device)
    _check(lib().ihs_gram(ctx._bind(), _p(SA), m, d, float(scale), _p(H)), "ihs_gram")
    return H


def ihs_small_step(A, b, spec: Spec, it: int, x, out=None, intermediates: bool = False, ctx: Context | None = None):
    """One OLS IHS iteration of a small dense problem in one launch (ihs.h);
    returns x_next, or (x_next, SA, g, H) with intermediates=True."""
    A = as_matrix(A)
    ctx = ctx or default_context(A.device)
    xn = out if out is not None else torch.empty_like(x)
    SA = _f64((spec.m, A.d), A.device) if intermediates else None
    g = _f64(A.d, A.device) if intermediates else None
    H = _f64((A.d, A.d), A.device) if intermediates else None
    mc, sp = A.c(), spec.c()
    _check(lib().ihs_small_step(ctx._bind(), C.byref(mc), _p(b), C.byref(sp), it, _p(x), _p(xn), _p(SA), _p(g),
                                _p(H)), "ihs_small_step")
    return (xn, SA, g, H) if intermediates else xn


# ------------------------------------------------------------------ a6
def ihs_gram_ols_update(SA: torch.Tensor, g, x, scale: float = 1.0, out=None, H=None, ctx: Context | None = None):
    """a4 + a6 for OLS: H = scale^2 SA^T SA, x_next = x + H^{-1} g; returns (x_next, H)."""
    ctx = ctx or default_context(SA.device)
    m, d = SA.shape
    xn = out if out is not None else torch.empty_like(x)
    H = H if H is not None else _f64((d, d), SA.device)
    _check(lib().ihs_gram_ols_update(ctx._bind(), _p(SA), m, d, float(scale), _p(g), _p(x), _p(xn), _p(H)),
           "ihs_gram_ols_update")
    return xn, H


def ihs_ols_update(H, g, x, out=None, ctx: Context | None = None):
    ctx = ctx or default_context(H.device)
    xn = out if out is not None else torch.empty_like(x)
    _check(lib().ihs_ols_update(ctx._bind(), _p(H), _p(g), x.numel(), _p(x), _p(xn)), "ihs_ols_update")
    ctx._release(H)
    return xn


def ihs_ols_factor(SA: torch.Tensor, scale: float = 1.0, out=None, ctx: Context | None = None):
    """Look-ahead OLS, part 1: Hinv = (scale^2 SA^T SA)^{-1} (d <= 128), computed on
    the context's factor stream after the work already on its stream.  Joined by
    the next ihs_ols_apply / ctx.synchronize(); read Hinv only after one of them."""
    ctx = ctx or default_context(SA.device)
    m, d = SA.shape
    Hinv = out if out is not None else _f64((d, d), SA.device)
    _check(lib().ihs_ols_factor(ctx._bind(), _p(SA), m, d, float(scale), _p(Hinv)), "ihs_ols_factor")
    ctx._hold(Hinv, SA)
    return Hinv


def ihs_gram_lookahead(SA: torch.Tensor, scale: float = 1.0, out=None, ctx: Context | None = None):
    """H = scale^2 SA^T SA on the context's factor stream (look-ahead Gram for the
    l1 / LASSO updates); joined by the next update that reads H / ctx.synchronize()."""
    ctx = ctx or default_context(SA.device)
    m, d = SA.shape
    H = out if out is not None else _f64((d, d), SA.device)
    _check(lib().ihs_gram_lookahead(ctx._bind(), _p(SA), m, d, float(scale), _p(H)), "ihs_gram_lookahead")
    ctx._hold(H, SA)
    return H


def ihs_ols_apply(Hinv, g, x, out=None, ctx: Context | None = None):
    """Look-ahead OLS, part 2: x_next = x + Hinv g (after the pending factor)."""
    ctx = ctx or default_context(Hinv.device)
    xn = out if out is not None else torch.empty_like(x)
    _check(lib().ihs_ols_apply(ctx._bind(), _p(Hinv), _p(g), x.numel(), _p(x), _p(xn)), "ihs_ols_apply")
    ctx._release(Hinv)
    return xn


def ihs_ols_lookahead_step(A, spec: Spec, it_next: int, b, x, Hinv, SA_next=None, Hinv_next=None, g=None,
                           out=None, ctx: Context | None = None):
    """One look-ahead OLS step on one rank (ihs.h): g at x, S^{it_next} A into
    SA_next and its factor into Hinv_next (both optional), x_next = x + Hinv g.
    Returns (x_next, g)."""
    A = as_matrix(A)
    ctx = ctx or default_context(A.device)
    g = g if g is not None else _f64(A.d, A.device)
    xn = out if out is not None else torch.empty_like(x)
    mc, sp = A.c(), spec.c()
    _check(lib().ihs_ols_lookahead_step(ctx._bind(), C.byref(mc), C.byref(sp), it_next, _p(b), _p(x), _p(Hinv),
                                        _p(SA_next), _p(Hinv_next), _p(g), _p(xn)), "ihs_ols_lookahead_step")
    ctx._release(Hinv)
    if Hinv_next is not None:
        ctx._hold(Hinv_next, SA_next)
    return xn, g


def inner_cfg(max_inner=20000, power_iters=50, inner_tol=1e-14, lip_safety=1.05, warm_power_iters=12) -> InnerCfg:
    return InnerCfg(max_inner, power_iters, inner_tol, lip_safety, warm_power_iters, 0)


def ihs_l1ball_update(H, g, x, radius, cfg: InnerCfg | None = None, out=None, inner=None,
                      ctx: Context | None = None):
    ctx = ctx or default_context(H.device)
    xn = out if out is not None else torch.empty_like(x)
    cfg = cfg or inner_cfg()
    _check(lib().ihs_l1ball_update(ctx._bind(), _p(H), _p(g), x.numel(), _p(x), float(radius), C.byref(cfg),
                                   _p(xn), _p(inner)), "ihs_l1ball_update")
    ctx._release(H)
    return xn


def ihs_lasso_update(H, g, x, lam, cfg: InnerCfg | None = None, out=None, inner=None,
                     ctx: Context | None = None):
    """NEXT-2: argmin_y 1/2 (y-x)^T H (y-x) - g^T (y-x) + lam ||y||_1."""
    ctx = ctx or default_context(H.device)
    xn = out if out is not None else torch.empty_like(x)
    cfg = cfg or inner_cfg()
    _check(lib().ihs_lasso_update(ctx._bind(), _p(H), _p(g), x.numel(), _p(x), float(lam), C.byref(cfg),
                                  _p(xn), _p(inner)), "ihs_lasso_update")
    ctx._release(H)
    return xn


# ------------------------------------------------------------------ a1-a7
def _solve(kind, A, b, spec, n_iters, iter0, x0, radius, cfg, trace, ctx, x_out, x_hist):
    A = A if isinstance(A, (Dense, Csr)) else as_matrix(A)
    dev = A.device
    ctx = ctx or default_context(dev if dev.type == "cuda" else None)
    d = A.d
    on_host = dev.type == "cpu"
    if x_out is None:
        x_out = torch.empty(d, dtype=torch.float64, device=dev, pin_memory=False)
    if x_hist is None:
        x_hist = torch.empty((n_iters + 1, d), dtype=torch.float64, device=dev)
    recs = (IterRecord * max(n_iters, 1))() if trace else None
    mc, sp = A.c(), spec.c()
    rp = C.cast(recs, C.POINTER(IterRecord)) if trace else None
    if kind == "ols":
        st = lib().ihs_solve_ols(ctx._bind(), C.byref(mc), _p(b), C.byref(sp), n_iters, iter0, _p(x0), _p(x_out),
                                 _p(x_hist), rp)
    else:
        c = cfg or inner_cfg()
        fn = lib().ihs_solve_lasso if kind == "lasso" else lib().ihs_solve_l1ball
        st = fn(ctx._bind(), C.byref(mc), _p(b), float(radius), C.byref(sp), n_iters, iter0, C.byref(c), _p(x0),
                _p(x_out), _p(x_hist), rp)
    if st not in (OK, ERR_NOT_CONVERGED):
        raise IhsError(st, f"ihs_solve_{kind}")
    out = {"x": x_out, "x_hist": x_hist, "status": st}
    if trace:
        out["trace"] = [dict(t_sketch_grad=r.t_sketch_grad, t_comm=r.t_comm, t_gram=r.t_gram, t_solve=r.t_solve,
                             inner_iters=r.inner_iters, status=r.status) for r in recs[:n_iters]]
    del on_host
    return out


def ihs_solve_ols(A, b, spec: Spec, n_iters: int, iter0: int = 0, x0=None, trace=False, ctx=None, x_out=None,
                  x_hist=None):
    """T IHS steps for OLS (Eq. (2), C = R^d).  A/b may live on the host (copied inside)."""
    return _solve("ols", A, b, spec, n_iters, iter0, x0, 0.0, None, trace, ctx, x_out, x_hist)


def ihs_solve_l1ball(A, b, radius: float, spec: Spec, n_iters: int, iter0: int = 0, cfg=None, x0=None,
                     trace=False, ctx=None, x_out=None, x_hist=None):
    """T IHS steps over {||x||_1 <= radius} with the PG inner solver."""
    return _solve("l1", A, b, spec, n_iters, iter0, x0, radius, cfg, trace, ctx, x_out, x_hist)


def ihs_solve_lasso(A, b, lam: float, spec: Spec, n_iters: int, iter0: int = 0, cfg=None, x0=None,
                    trace=False, ctx=None, x_out=None, x_hist=None):
    """NEXT-2: T IHS steps for 1/2||Ax-b||^2 + lam ||x||_1 (penalty kept in every step)."""
    return _solve("lasso", A, b, spec, n_iters, iter0, x0, lam, cfg, trace, ctx, x_out, x_hist)


def ihs_pred_err2(A, X: torch.Tensor, xref: torch.Tensor, ctx: Context | None = None):
    """(err2[k] = ||A(X[k]-xref)||^2, ref2 = ||A xref||^2) on the device (a7)."""
    A = as_matrix(A)
    ctx = ctx or default_context(A.device)
    X = X.reshape(-1, A.d).contiguous()
    err2 = _f64(max(X.shape[0], 1), A.device)
    ref2 = _f64(1, A.device)
    mc = A.c()
    _check(lib().ihs_pred_err2(ctx._bind(), C.byref(mc), _p(X), X.shape[0], _p(xref), _p(err2), _p(ref2)),
           "ihs_pred_err2")
    return err2[: X.shape[0]], ref2
