"""CPU ORACLE — TEST INFRASTRUCTURE, NOT PRODUCT CODE.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) may import this package.  The product package
``paper_2503_04914_b200`` never imports it and shares no code with it.

* ``msk_oracle.c`` (loaded through ctypes as ``liboracle.so``): the plain C
  FP64 reference of the sequential multiscale method, patterns, CG,
  evaluation and the literal monolithic Jacobi (see its header).
* ``dense.py``: dense numpy forms of T_L, T'_L, M, the thresholded M~(T) and
  the Figures 1-3 quantities (small hierarchies only).

Parity unpinned: none of the exported functions — every one is pinned by a
``tests/test_oracle_*.py`` check against the paper.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "msk_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

_dp = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (-O2, no FMA contraction, reading C-4)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
               "-o", _LIB, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


NATIVE_FLAGS = ["-O3", "-march=native", "-ffp-contract=off", "-fno-fast-math", "-fopenmp"]


def build_native() -> str:
    """The same source for the CPU baseline: -O3 -march=native -ffp-contract=off
    -fopenmp, compiled for THIS host into the temp directory (never shipped:
    -march=native code may not run on another CPU).  Results are bit-identical
    to build()'s library for any thread count (test_oracle_solvers.py)."""
    import hashlib
    import tempfile
    with open(_SRC, "rb") as fh:
        tag = hashlib.sha1(fh.read() + " ".join(NATIVE_FLAGS).encode()).hexdigest()[:12]
    path = os.path.join(tempfile.gettempdir(), f"msk_oracle_native_{tag}_{os.getpid()}.so")
    if not os.path.exists(path):
        subprocess.check_call(["gcc"] + NATIVE_FLAGS + ["-fPIC", "-shared", "-o", path, _SRC, "-lm"])
    return path


def use_native(threads: int = 1) -> int:
    """Switch this process's oracle calls to the native (-O3 -march=native
    -fopenmp) build with `threads` OpenMP threads; returns the threads in
    effect.  use_plain() switches back."""
    global _lib
    _lib = _load(build_native())
    return int(_lib.mo_set_threads(int(threads)))


def use_plain() -> None:
    global _lib
    _lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = _load(build())
    return _lib


def _load(path):
    if True:
        L = ctypes.CDLL(path)
        L.mo_phi.restype = ctypes.c_double
        L.mo_phi.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double]
        L.mo_kernel.restype = ctypes.c_double
        L.mo_kernel.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double, _dp, _dp]
        for name in ("mo_pattern_bruteforce", "mo_pattern_grid"):
            fn = getattr(L, name)
            fn.restype = ctypes.c_int64
            fn.argtypes = [ctypes.c_int, ctypes.c_int64, _dp, ctypes.c_int64, _dp,
                           ctypes.c_double, _i64p, _i32p]
        L.mo_values.restype = None
        L.mo_values.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_int64,
                                _dp, _dp, _i64p, _i32p, _dp]
        L.mo_spmv.restype = None
        L.mo_spmv.argtypes = [ctypes.c_int64, _i64p, _i32p, _dp, _dp, _dp]
        L.mo_apply.restype = ctypes.c_int
        L.mo_apply.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_int64, _dp,
                               ctypes.c_int64, _dp, _dp, _dp]
        L.mo_cg.restype = ctypes.c_int
        L.mo_cg.argtypes = [ctypes.c_int64, _i64p, _i32p, _dp, _dp, _dp, ctypes.c_double,
                            ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
        L.mo_cholesky_solve.restype = ctypes.c_int
        L.mo_cholesky_solve.argtypes = [ctypes.c_int64, _i64p, _i32p, _dp, _dp, _dp]
        pp = ctypes.POINTER(_dp)
        L.mo_sequential.restype = ctypes.c_int
        L.mo_sequential.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _i64p, pp, _dp, pp,
                                    ctypes.c_double, ctypes.c_int, ctypes.c_int64, pp,
                                    ctypes.POINTER(ctypes.c_int), _dp]
        L.mo_evaluate.restype = ctypes.c_int
        L.mo_evaluate.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _i64p, pp, _dp, pp,
                                  ctypes.c_int64, _dp, _dp]
        L.mo_jacobi_literal.restype = ctypes.c_int
        L.mo_jacobi_literal.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _i64p, pp, _dp,
                                        pp, pp, ctypes.c_double, ctypes.c_double, ctypes.c_int,
                                        ctypes.c_int64, pp, pp]
        L.mo_thresholded.restype = ctypes.c_int
        L.mo_thresholded.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _i64p, pp, _dp, _dp,
                                     ctypes.c_double, pp, pp, pp, _i64p]
        L.mo_separation.restype = ctypes.c_double
        L.mo_separation.argtypes = [ctypes.c_int, ctypes.c_int64, _dp]
        L.mo_mas_row_residual.restype = ctypes.c_double
        L.mo_mas_row_residual.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _i64p, pp, _dp,
                                          pp, ctypes.c_double, ctypes.c_int64, _dp]
        L.mo_set_threads.restype = ctypes.c_int
        L.mo_set_threads.argtypes = [ctypes.c_int]
    return L


# ---------------------------------------------------------------------------
# numpy-friendly wrappers
# ---------------------------------------------------------------------------
def _c(a, dt=np.float64):
    return np.ascontiguousarray(a, dtype=dt)


def _ptr(a, t=_dp):
    return a.ctypes.data_as(t)


def _ptrs(arrays):
    arr = (_dp * len(arrays))(*[_ptr(a) for a in arrays])
    return ctypes.cast(arr, ctypes.POINTER(_dp)), arr


def phi(d, k, r):
    return lib().mo_phi(d, k, float(r))


def kernel(d, k, delta, x, y):
    x, y = _c(x), _c(y)
    return lib().mo_kernel(d, k, float(delta), _ptr(x), _ptr(y))


def pattern(X, Y, delta, method="grid"):
    """CSR pattern (row_ptr int64, col int32 ascending) of r^2 < delta^2."""
    X, Y = _c(X), _c(Y)
    d = X.shape[1]
    nr, nc = X.shape[0], Y.shape[0]
    fn = lib().mo_pattern_grid if method == "grid" else lib().mo_pattern_bruteforce
    rp = np.zeros(nr + 1, dtype=np.int64)
    nnz = fn(d, nr, _ptr(X), nc, _ptr(Y), float(delta), _ptr(rp, _i64p), None)
    if nnz < 0:
        raise MemoryError("oracle pattern allocation failed")
    col = np.zeros(max(nnz, 1), dtype=np.int32)
    fn(d, nr, _ptr(X), nc, _ptr(Y), float(delta), _ptr(rp, _i64p), _ptr(col, _i32p))
    return rp, col[:nnz]


def block(X, Y, delta, k=1, method="grid"):
    """(row_ptr, col, val) of B = (Phi_delta(x_j - y_n)) in CSR."""
    X, Y = _c(X), _c(Y)
    rp, col = pattern(X, Y, delta, method)
    val = np.zeros(max(len(col), 1))
    colc = _c(col if len(col) else np.zeros(1, np.int32), np.int32)
    lib().mo_values(X.shape[1], k, float(delta), X.shape[0], _ptr(X), _ptr(Y),
                    _ptr(rp, _i64p), _ptr(colc, _i32p), _ptr(val))
    return rp, col, val[:len(col)]


def spmv(rp, col, val, v):
    v = _c(v)
    n = len(rp) - 1
    y = np.zeros(n)
    colc = _c(col if len(col) else np.zeros(1, np.int32), np.int32)
    valc = _c(val if len(val) else np.zeros(1))
    lib().mo_spmv(n, _ptr(_c(rp, np.int64), _i64p), _ptr(colc, _i32p), _ptr(valc), _ptr(v), _ptr(y))
    return y


def apply(X, Y, delta, v, k=1):
    X, Y, v = _c(X), _c(Y), _c(v)
    out = np.zeros(X.shape[0])
    if lib().mo_apply(X.shape[1], k, float(delta), X.shape[0], _ptr(X), Y.shape[0], _ptr(Y),
                      _ptr(v), _ptr(out)):
        raise MemoryError
    return out


def cg(rp, col, val, b, tol, max_iter=20000):
    b = _c(b)
    n = len(rp) - 1
    x = np.zeros(n)
    it = ctypes.c_int(0)
    colc = _c(col, np.int32)
    st = lib().mo_cg(n, _ptr(_c(rp, np.int64), _i64p), _ptr(colc, _i32p), _ptr(_c(val)), _ptr(b),
                     _ptr(x), float(tol), int(max_iter), ctypes.byref(it))
    return x, it.value, st


def cholesky_solve(rp, col, val, b):
    b = _c(b)
    n = len(rp) - 1
    x = np.zeros(n)
    st = lib().mo_cholesky_solve(n, _ptr(_c(rp, np.int64), _i64p), _ptr(_c(col, np.int32), _i32p),
                                 _ptr(_c(val)), _ptr(b), _ptr(x))
    if st:
        raise np.linalg.LinAlgError(f"cholesky failed ({st})")
    return x


def _hier_args(points, delta):
    pts = [_c(p) for p in points]
    d = pts[0].shape[1]
    n = np.array([p.shape[0] for p in pts], dtype=np.int64)
    return pts, d, n, _c(delta)


def sequential(points, delta, f, tol=1e-12, k=1, max_iter=20000, direct_max_n=4000, count=True):
    """eq:mas level by level (O4). Returns (alpha list, iters list, counters)."""
    pts, d, n, dl = _hier_args(points, delta)
    fs = [_c(x) for x in f]
    alpha = [np.zeros(int(m)) for m in n]
    iters = (ctypes.c_int * len(pts))()
    counters = np.zeros(3)
    pp, _k1 = _ptrs(pts)
    fp, _k2 = _ptrs(fs)
    ap, _k3 = _ptrs(alpha)
    st = lib().mo_sequential(d, k, len(pts), _ptr(n, _i64p), pp, _ptr(dl), fp, float(tol),
                             int(max_iter), int(direct_max_n), ap, iters,
                             _ptr(counters) if count else None)
    if st:
        raise RuntimeError(f"oracle sequential solve failed ({st})")
    return alpha, list(iters), counters


def evaluate(points, delta, alpha, x, k=1):
    """f_L(x), eq:fapproximation (O5)."""
    pts, d, n, dl = _hier_args(points, delta)
    al = [_c(a) for a in alpha]
    x = _c(x)
    s = np.zeros(x.shape[0])
    pp, _k1 = _ptrs(pts)
    ap, _k2 = _ptrs(al)
    if lib().mo_evaluate(d, k, len(pts), _ptr(n, _i64p), pp, _ptr(dl), ap, x.shape[0],
                         _ptr(x), _ptr(s)):
        raise MemoryError
    return s


def jacobi_literal(points, delta, f, tol=1e-12, inner_tol=None, beta0=None, k=1,
                   max_iter=20000, direct_max_n=4000):
    """Literal Algorithm 2 + block CG (O6). Returns (alpha, beta)."""
    pts, d, n, dl = _hier_args(points, delta)
    fs = [_c(x) for x in f]
    alpha = [np.zeros(int(m)) for m in n]
    beta = [np.zeros(int(m)) for m in n]
    pp, _k1 = _ptrs(pts)
    fp, _k2 = _ptrs(fs)
    ap, _k3 = _ptrs(alpha)
    bp, _k4 = _ptrs(beta)
    if beta0 is not None:
        b0 = [_c(x) for x in beta0]
        b0p, _k5 = _ptrs(b0)
    else:
        b0p = None
    st = lib().mo_jacobi_literal(d, k, len(pts), _ptr(n, _i64p), pp, _ptr(dl), fp, b0p,
                                 float(tol), float(inner_tol if inner_tol else tol / 10),
                                 int(max_iter), int(direct_max_n), bp, ap)
    if st:
        raise RuntimeError(f"oracle jacobi failed ({st})")
    return alpha, beta


def thresholded(points, delta, q, T, f, k=1):
    """O7: forward substitution with M~(T) + block solves. Returns (alpha, beta, nnz)."""
    pts, d, n, dl = _hier_args(points, delta)
    qq = _c(q)
    fs = [_c(x) for x in f]
    alpha = [np.zeros(int(m)) for m in n]
    beta = [np.zeros(int(m)) for m in n]
    pp, _k1 = _ptrs(pts)
    fp, _k2 = _ptrs(fs)
    ap, _k3 = _ptrs(alpha)
    bp, _k4 = _ptrs(beta)
    nnz = np.zeros(1, dtype=np.int64)
    st = lib().mo_thresholded(d, k, len(pts), _ptr(n, _i64p), pp, _ptr(dl), _ptr(qq), float(T), fp, bp, ap,
                              _ptr(nnz, _i64p))
    if st:
        raise RuntimeError(f"oracle thresholded solve failed ({st})")
    return alpha, beta, int(nnz[0])


def separation(P):
    P = _c(P)
    return lib().mo_separation(P.shape[1], P.shape[0], _ptr(P))


def mas_row_residual(points, delta, alpha, level, j, f_j, k=1):
    """Row j of eq:mas at level `level` by brute force: (residual, abs scale)."""
    pts, d, n, dl = _hier_args(points, delta)
    al = [_c(a) for a in alpha]
    pp, _k1 = _ptrs(pts)
    ap, _k2 = _ptrs(al)
    scale = ctypes.c_double(0.0)
    r = lib().mo_mas_row_residual(d, k, int(level), _ptr(n, _i64p), pp, _ptr(dl), ap,
                                  float(f_j), int(j), ctypes.byref(scale))
    return r, scale.value
