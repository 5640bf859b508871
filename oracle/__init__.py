"""CPU oracle for the IHS hot path of arXiv 1910.14166 -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
``paper_1910_14166_b200`` never imports it, and it never imports the product.

The arithmetic lives in ``oracle/ihs_oracle.c`` (plain sequential C, fp64,
``-O2 -ffp-contract=off``); this module only marshals numpy arrays through
ctypes.  Each wrapper names the PAPER.md passage its C function follows.

Pinned by ``tests/test_oracle_*.py`` (see DESIGN.md section 4 for the pin of
every function).  No function here is "parity unpinned".
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ihs_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

OK, ERR_INVALID, ERR_NOT_SPD, ERR_NOT_CONVERGED = 0, 1, 3, 4


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain C, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11",
                               "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_SRC_OMP = os.path.join(_HERE, "ihs_oracle_omp.c")
_LIB_OMP = os.path.join(_HERE, "liboracle_omp.so")
_lib_omp = None


def build_omp(force: bool = False) -> str:
    """liboracle_omp.so: the OpenMP timing variants of the row-parallel phases."""
    if force or not os.path.exists(_LIB_OMP) or os.path.getmtime(_LIB_OMP) < os.path.getmtime(_SRC_OMP):
        tmp = _LIB_OMP + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11", "-fopenmp",
                               "-fPIC", "-shared", "-o", tmp, _SRC_OMP, "-lm"])
        os.replace(tmp, _LIB_OMP)
    return _LIB_OMP


def lib_omp():
    global _lib_omp
    with _lock:
        if _lib_omp is None:
            build_omp()
            L = C.CDLL(_LIB_OMP)
            i64, i32, u64, p = C.c_int64, C.c_int32, C.c_uint64, C.c_void_p
            L.or_omp_threads.restype = C.c_int
            L.or_omp_threads.argtypes = []
            L.or_sketch_dense_omp.restype = None
            L.or_sketch_dense_omp.argtypes = [i64, i64, p, i64, u64, u64, i64, i32, p]
            L.or_grad_dense_omp.restype = None
            L.or_grad_dense_omp.argtypes = [i64, i64, p, p, p, p]
            _lib_omp = L
    return _lib_omp


def omp_threads() -> int:
    return int(lib_omp().or_omp_threads())


def sketch_dense_omp(A, seed, t, m, s, row_offset=0):
    """OpenMP timing variant of sketch_dense (row blocks per thread, partials
    added in thread order; equal to it up to rounding)."""
    A = _f64(A)
    n, d = A.shape
    SA = np.empty((m, d))
    lib_omp().or_sketch_dense_omp(n, d, _ptr(A), row_offset, seed, t, m, s, _ptr(SA))
    return SA


def grad_dense_omp(A, b, x):
    """OpenMP timing variant of grad_dense."""
    A, b, x = _f64(A), _f64(b), _f64(x)
    g = np.empty(A.shape[1])
    lib_omp().or_grad_dense_omp(A.shape[0], A.shape[1], _ptr(A), _ptr(b), _ptr(x), _ptr(g))
    return g


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(_LIB)
            i64, i32, u64, dbl, p = C.c_int64, C.c_int32, C.c_uint64, C.c_double, C.c_void_p
            sig = {
                "or_splitmix64": (u64, [u64]),
                "or_iter_key": (u64, [u64, u64]),
                "or_hash_rows": (None, [u64, u64, i32, i64, i64, i64, p, p]),
                "or_sketch_dense_hs": (None, [i64, i64, p, i64, i32, p, p, p]),
                "or_sketch_dense": (None, [i64, i64, p, i64, u64, u64, i64, i32, p]),
                "or_sketch_dense_rows": (None, [i64, i64, p, i64, u64, u64, i64, i32, i64, p, p]),
                "or_sketch_csr": (None, [i64, i64, p, p, p, i64, u64, u64, i64, i32, p]),
                "or_grad_dense": (None, [i64, i64, p, p, p, p]),
                "or_grad_csr": (None, [i64, i64, p, p, p, p, p, p]),
                "or_matvec_dense": (None, [i64, i64, p, p, p]),
                "or_matvec_csr": (None, [i64, p, p, p, p, p]),
                "or_gram": (None, [i64, i64, p, p]),
                "or_cholesky": (C.c_int, [i64, p, p]),
                "or_chol_solve": (None, [i64, p, p, p]),
                "or_ols_step": (C.c_int, [i64, p, p, p, p]),
                "or_project_l1": (None, [i64, p, dbl, p]),
                "or_power_lmax": (dbl, [i64, p, i32]),
                "or_l1ball_step": (C.c_int, [i64, p, p, p, dbl, i32, dbl, i32, dbl, p, p]),
                "or_lasso_step": (C.c_int, [i64, p, p, p, dbl, i32, dbl, i32, dbl, p, p]),
                "or_ihs_solve": (C.c_int, [i32, i64, i64, p, p, p, p, u64, i64, i32, i32, u64,
                                           i32, dbl, i32, dbl, i32, dbl, p, p, p]),
                "or_normal_dense": (None, [i64, i64, p, p, p, p]),
                "or_exact_ols": (C.c_int, [i32, i64, i64, p, p, p, p, p]),
                "or_exact_l1ball": (C.c_int, [i32, i64, i64, p, p, p, p, dbl, i32, i32, dbl, p]),
                "or_exact_lasso": (C.c_int, [i64, i64, p, p, dbl, i32, i32, dbl, p]),
                "or_pred_rel_err": (dbl, [i32, i64, i64, p, p, p, p, p]),
            }
            for name, (res, args) in sig.items():
                f = getattr(L, name)
                f.restype = res
                f.argtypes = args
            _lib = L
    return _lib


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class OracleError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"oracle {what}: status {status}")
        self.status = status


# ---------------------------------------------------------------- hash (a1)
def splitmix64(x: int) -> int:
    """splitmix64 step (R1): golden-gamma add + finaliser."""
    return int(lib().or_splitmix64(C.c_uint64(x & 0xFFFFFFFFFFFFFFFF)))


def iter_key(seed: int, t: int) -> int:
    """k_t = SM(SM(seed) ^ t)  (R1, R2)."""
    return int(lib().or_iter_key(seed, t))


def hash_rows(seed: int, t: int, m: int, s: int, row_begin: int, count: int):
    """Buckets/signs of rows [row_begin, row_begin+count), shape (count, s).
    CountSketch / SJLT construction, PAPER.md:175-184 (section 2)."""
    b = np.empty((count, s), np.int32)
    g = np.empty((count, s), np.int8)
    lib().or_hash_rows(seed, t, s, m, row_begin, count, _ptr(b), _ptr(g))
    return b, g


# -------------------------------------------------------------- sketch (a2)
def sketch_dense_hs(A, m: int, bucket, sign):
    """SA from explicit (h, sigma) arrays of shape (n, s) -- PAPER.md:175-184, 236-240."""
    A = _f64(A)
    n, d = A.shape
    bucket = np.ascontiguousarray(bucket, np.int32).reshape(n, -1)
    sign = np.ascontiguousarray(sign, np.int8).reshape(n, -1)
    s = bucket.shape[1]
    SA = np.empty((m, d))
    lib().or_sketch_dense_hs(n, d, _ptr(A), m, s, _ptr(bucket), _ptr(sign), _ptr(SA))
    return SA


def sketch_dense(A, seed: int, t: int, m: int, s: int = 1, row_offset: int = 0):
    """Hash-defined SA for a dense row block starting at global row row_offset."""
    A = _f64(A)
    n, d = A.shape
    SA = np.empty((m, d))
    lib().or_sketch_dense(n, d, _ptr(A), row_offset, seed, t, m, s, _ptr(SA))
    return SA


def sketch_dense_rows(A, seed: int, t: int, m: int, s: int, rows, row_offset: int = 0):
    """Only the SA rows listed in ``rows`` (sampled outputs at full size)."""
    A = _f64(A)
    n, d = A.shape
    rows = np.ascontiguousarray(rows, np.int64)
    out = np.empty((rows.size, d))
    lib().or_sketch_dense_rows(n, d, _ptr(A), row_offset, seed, t, m, s, rows.size, _ptr(rows), _ptr(out))
    return out


def sketch_csr(row_ptr, col, val, d: int, seed: int, t: int, m: int, s: int = 1, row_offset: int = 0):
    row_ptr = np.ascontiguousarray(row_ptr, np.int64)
    col = np.ascontiguousarray(col, np.int32)
    val = _f64(val)
    n = row_ptr.size - 1
    SA = np.empty((m, d))
    lib().or_sketch_csr(n, d, _ptr(row_ptr), _ptr(col), _ptr(val), row_offset, seed, t, m, s, _ptr(SA))
    return SA


# ------------------------------------------------------------ gradient (a5)
def grad_dense(A, b, x):
    """g = A^T (b - A x)  (Eq. (2) linear term; sign R21)."""
    A, b, x = _f64(A), _f64(b), _f64(x)
    n, d = A.shape
    g = np.empty(d)
    lib().or_grad_dense(n, d, _ptr(A), _ptr(b), _ptr(x), _ptr(g))
    return g


def grad_csr(row_ptr, col, val, d: int, b, x):
    row_ptr = np.ascontiguousarray(row_ptr, np.int64)
    col = np.ascontiguousarray(col, np.int32)
    val, b, x = _f64(val), _f64(b), _f64(x)
    g = np.empty(d)
    lib().or_grad_csr(row_ptr.size - 1, d, _ptr(row_ptr), _ptr(col), _ptr(val), _ptr(b), _ptr(x), _ptr(g))
    return g


def matvec_dense(A, x):
    A, x = _f64(A), _f64(x)
    y = np.empty(A.shape[0])
    lib().or_matvec_dense(A.shape[0], A.shape[1], _ptr(A), _ptr(x), _ptr(y))
    return y


def matvec_csr(row_ptr, col, val, x):
    row_ptr = np.ascontiguousarray(row_ptr, np.int64)
    col = np.ascontiguousarray(col, np.int32)
    val, x = _f64(val), _f64(x)
    y = np.empty(row_ptr.size - 1)
    lib().or_matvec_csr(row_ptr.size - 1, _ptr(row_ptr), _ptr(col), _ptr(val), _ptr(x), _ptr(y))
    return y


# ---------------------------------------------------------------- Gram (a4)
def gram(SA):
    """H = (SA)^T SA (approximate Hessian)."""
    SA = _f64(SA)
    m, d = SA.shape
    H = np.empty((d, d))
    lib().or_gram(m, d, _ptr(SA), _ptr(H))
    return H


# ---------------------------------------------------------- inner QP (a6)
def cholesky(H):
    H = _f64(H)
    d = H.shape[0]
    L = np.empty((d, d))
    st = lib().or_cholesky(d, _ptr(H), _ptr(L))
    if st != OK:
        raise OracleError(st, "cholesky")
    return L


def chol_solve(L, g):
    L, g = _f64(L), _f64(g)
    u = np.empty(L.shape[0])
    lib().or_chol_solve(L.shape[0], _ptr(L), _ptr(g), _ptr(u))
    return u


def ols_step(H, g, x):
    """x^{t+1} = x^t + H^{-1} g  (Eq. (2) with C = R^d)."""
    H, g, x = _f64(H), _f64(g), _f64(x)
    xn = np.empty_like(x)
    st = lib().or_ols_step(H.shape[0], _ptr(H), _ptr(g), _ptr(x), _ptr(xn))
    if st != OK:
        raise OracleError(st, "ols_step")
    return xn


def project_l1(v, tau: float):
    """Euclidean projection onto {||x||_1 <= tau} (reading R8)."""
    v = _f64(v)
    out = np.empty_like(v)
    lib().or_project_l1(v.size, _ptr(v), float(tau), _ptr(out))
    return out


def power_lmax(H, iters: int = 50) -> float:
    H = _f64(H)
    return float(lib().or_power_lmax(H.shape[0], _ptr(H), iters))


def l1ball_step(H, g, x, tau, max_inner=20000, tol=1e-14, power_iters=50, safety=1.05):
    """Projected-gradient solve of Eq. (2) over the l1 ball (reading R10).
    Returns (x_next, inner_iterations, status)."""
    H, g, x = _f64(H), _f64(g), _f64(x)
    xn = np.empty_like(x)
    it = C.c_int32(0)
    st = lib().or_l1ball_step(H.shape[0], _ptr(H), _ptr(g), _ptr(x), float(tau), max_inner, tol,
                              power_iters, safety, _ptr(xn), C.byref(it))
    return xn, int(it.value), int(st)


def lasso_step(H, g, x, lam, max_inner=20000, tol=1e-14, power_iters=50, safety=1.05):
    """NEXT-2: proximal-gradient solve of Eq. (2) + lambda ||x||_1 (readings R10, R23).
    Returns (x_next, inner_iterations, status)."""
    H, g, x = _f64(H), _f64(g), _f64(x)
    xn = np.empty_like(x)
    it = C.c_int32(0)
    st = lib().or_lasso_step(H.shape[0], _ptr(H), _ptr(g), _ptr(x), float(lam), max_inner, tol,
                             power_iters, safety, _ptr(xn), C.byref(it))
    return xn, int(it.value), int(st)


# ------------------------------------------------------------ IHS (a1-a7)
def ihs_solve(A=None, b=None, *, csr=None, d=None, seed=0, m, s=1, T, iter0=0,
              constraint="ols", tau=0.0, max_inner=20000, tol=1e-14, power_iters=50,
              safety=1.05, x0=None):
    """Run T IHS steps (Eq. (2)); returns (x_hist (T+1, d), inner_iters (T,)).
    ``csr`` = (row_ptr, col, val) selects the CSR layout."""
    b = _f64(b)
    if csr is None:
        A = _f64(A)
        n, d = A.shape
        layout, vals, rp, cl = 0, A, None, None
    else:
        rp = np.ascontiguousarray(csr[0], np.int64)
        cl = np.ascontiguousarray(csr[1], np.int32)
        vals = _f64(csr[2])
        n, layout = rp.size - 1, 1
    xh = np.empty((T + 1, d))
    inner = np.zeros(max(T, 1), np.int32)
    x0a = None if x0 is None else _f64(x0)
    st = lib().or_ihs_solve(layout, n, d, _ptr(vals), _ptr(rp), _ptr(cl), _ptr(b), seed, m, s, T, iter0,
                            {"ols": 0, "l1ball": 1, "lasso": 2}[constraint], float(tau), max_inner, tol,
                            power_iters,
                            safety, _ptr(x0a), _ptr(xh), _ptr(inner))
    if st != OK:
        raise OracleError(st, "ihs_solve")
    return xh, inner[:T]


def exact_ols(A=None, b=None, *, csr=None, d=None):
    """x_OPT of Eq. (1) with C = R^d: normal equations + one refinement step (O10)."""
    b = _f64(b)
    if csr is None:
        A = _f64(A)
        n, d = A.shape
        layout, vals, rp, cl = 0, A, None, None
    else:
        rp = np.ascontiguousarray(csr[0], np.int64)
        cl = np.ascontiguousarray(csr[1], np.int32)
        vals = _f64(csr[2])
        n, layout = rp.size - 1, 1
    x = np.empty(d)
    st = lib().or_exact_ols(layout, n, d, _ptr(vals), _ptr(rp), _ptr(cl), _ptr(b), _ptr(x))
    if st != OK:
        raise OracleError(st, "exact_ols")
    return x


def exact_l1ball(A, b, tau, outer=8, max_inner=200000, tol=1e-15):
    """x_OPT over {||x||_1 <= tau}: PG with the exact Hessian A^T A (O10)."""
    A, b = _f64(A), _f64(b)
    n, d = A.shape
    x = np.empty(d)
    st = lib().or_exact_l1ball(0, n, d, _ptr(A), None, None, _ptr(b), float(tau), outer, max_inner, tol, _ptr(x))
    if st != OK:
        raise OracleError(st, "exact_l1ball")
    return x


def exact_lasso(A, b, lam, outer=8, max_inner=200000, tol=1e-15):
    """NEXT-2: x_OPT of 1/2||Ax - b||^2 + lam ||x||_1: IHS with A^T A."""
    A, b = _f64(A), _f64(b)
    n, d = A.shape
    x = np.empty(d)
    st = lib().or_exact_lasso(n, d, _ptr(A), _ptr(b), float(lam), outer, max_inner, tol, _ptr(x))
    if st != OK:
        raise OracleError(st, "exact_lasso")
    return x


def pred_rel_err(x, xref, A=None, *, csr=None, d=None):
    """||A(x - xref)||_2 / ||A xref||_2."""
    x, xref = _f64(x), _f64(xref)
    if csr is None:
        A = _f64(A)
        n, d = A.shape
        return float(lib().or_pred_rel_err(0, n, d, _ptr(A), None, None, _ptr(x), _ptr(xref)))
    rp = np.ascontiguousarray(csr[0], np.int64)
    cl = np.ascontiguousarray(csr[1], np.int32)
    vals = _f64(csr[2])
    return float(lib().or_pred_rel_err(1, rp.size - 1, d, _ptr(vals), _ptr(rp), _ptr(cl), _ptr(x), _ptr(xref)))
