"""CPU oracle for G_RIP construction and cutsize -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product package ``paper_1710_07769_b200`` never imports it.

Thin ctypes marshalling over ``rig_oracle.c`` (every arithmetic step lives in
that file, with its PAPER.md citation).  Pins: ``tests/test_oracle_pins.py``.
Parity pinned for: scaling, transpose, products, build (structure, values,
diag, nnz(C)), cutsize, inter-block inner-product matrix and part weights
(SURVEY.md §8(f) f2), dense-column sparsification and integer edge weights
(f1).  Unpinned: nothing the build path uses; the paper's
12x12 sample is in a missing figure and is not
reproduced.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "rig_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared", "-std=gnu99"]


def default_threads() -> int:
    """Host cores this process may use (os.sched_getaffinity), capped at 64."""
    try:
        return max(1, min(64, len(os.sched_getaffinity(0))))
    except Exception:
        return max(1, min(64, os.cpu_count() or 1))


def build_lib(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".{os.getpid()}.tmp"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build_lib())
        i64, i32, p = ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p
        _lib.orc_scale_rows.argtypes = [i64, p, p, p, p]
        _lib.orc_transpose.argtypes = [i64, i64, p, p, p, p, p, p]
        _lib.orc_row_products.argtypes = [i64, p, p, p, p]
        _lib.orc_row_products.restype = i64
        _lib.orc_build.argtypes = [i64, i64, p, p, p, p, p, p, ctypes.c_double, i64, i64,
                                   p, p, p, p, p, p]
        _lib.orc_free.argtypes = [p]
        _lib.orc_build_par.argtypes = [i64, i64, p, p, p, p, p, p, ctypes.c_double, i64, i64, ctypes.c_int,
                                       p, p, p, p, p, p]
        _lib.orc_cutsize.argtypes = [i64, i64, p, p, p, i64, p, i32, p, p, p]
        _lib.orc_ip_matrix.argtypes = [i64, i64, p, p, p, i64, p, i32, p, p, p]
        _lib.orc_dense_threshold.argtypes = [i64]
        _lib.orc_dense_threshold.restype = i64
        _lib.orc_sparsify.argtypes = [i64, i64, p, p, p, p, p, p, p]
        _lib.orc_int_weights.argtypes = [i64, p, i64, p]
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code, what):
        super().__init__(f"oracle {what} failed with status {code}")
        self.code = code


ORC_ERR_INVALID, ORC_ERR_ZERO_ROW, ORC_ERR_NONFINITE, ORC_ERR_NOMEM = -1, -3, -4, -5


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def scale(row_ptr, val):
    row_ptr, val = _c(row_ptr, np.int64), _c(val, np.float64)
    n = row_ptr.size - 1
    out = np.empty_like(val)
    norms = np.empty(n, dtype=np.float64)
    st = lib().orc_scale_rows(n, _p(row_ptr), _p(val), _p(out), _p(norms))
    if st:
        raise OracleError(st, "scale_rows")
    return out, norms


def transpose(nrows, ncols, row_ptr, col_idx, val):
    row_ptr, col_idx, val = _c(row_ptr, np.int64), _c(col_idx, np.int32), _c(val, np.float64)
    nnz = int(row_ptr[-1])
    col_ptr = np.empty(ncols + 1, dtype=np.int64)
    row_idx = np.empty(nnz, dtype=np.int32)
    valT = np.empty(nnz, dtype=np.float64)
    st = lib().orc_transpose(nrows, ncols, _p(row_ptr), _p(col_idx), _p(val), _p(col_ptr),
                             _p(row_idx), _p(valT))
    if st:
        raise OracleError(st, "transpose")
    return col_ptr, row_idx, valT


def row_products(row_ptr, col_idx, col_ptr):
    row_ptr, col_idx, col_ptr = _c(row_ptr, np.int64), _c(col_idx, np.int32), _c(col_ptr, np.int64)
    n = row_ptr.size - 1
    f = np.empty(n, dtype=np.int64)
    total = lib().orc_row_products(n, _p(row_ptr), _p(col_idx), _p(col_ptr), _p(f))
    return f, int(total)


class Graph:
    """Oracle output for rows [row_begin, row_end)."""

    def __init__(self, row_ptr, col, w, diag, nnzc, row_begin, products, a_hat=None, csc=None):
        self.row_ptr, self.col, self.w, self.diag, self.nnzc = row_ptr, col, w, diag, nnzc
        self.row_begin = row_begin
        self.products = products
        self.a_hat = a_hat
        self.csc = csc

    @property
    def nnz(self):
        return int(self.row_ptr[-1])


def build_from_scaled(nrows, ncols, row_ptr, col_idx, val_hat, csc, drop_tol, row_begin=0, row_end=None,
                      threads=1):
    """Rows [row_begin, row_end) of G_RIP; threads > 1 runs row chunks of the
    same C routine concurrently (orc_build_par): identical output."""
    row_ptr, col_idx, val_hat = _c(row_ptr, np.int64), _c(col_idx, np.int32), _c(val_hat, np.float64)
    col_ptr, row_idx, valT = csc
    row_end = nrows if row_end is None else row_end
    nloc = row_end - row_begin
    L = lib()
    rp, gc, gw = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
    gnnz = ctypes.c_int64()
    diag = np.empty(nloc, dtype=np.float64)
    nnzc = np.empty(nloc, dtype=np.int64)
    if threads > 1:
        st = L.orc_build_par(nrows, ncols, _p(row_ptr), _p(col_idx), _p(val_hat), _p(col_ptr), _p(row_idx),
                             _p(valT), float(drop_tol), row_begin, row_end, int(threads), ctypes.byref(rp),
                             ctypes.byref(gc), ctypes.byref(gw), ctypes.byref(gnnz), _p(diag), _p(nnzc))
    else:
        st = L.orc_build(nrows, ncols, _p(row_ptr), _p(col_idx), _p(val_hat), _p(col_ptr), _p(row_idx),
                         _p(valT), float(drop_tol), row_begin, row_end, ctypes.byref(rp), ctypes.byref(gc),
                         ctypes.byref(gw), ctypes.byref(gnnz), _p(diag), _p(nnzc))
    if st:
        raise OracleError(st, "build")
    g = gnnz.value
    try:
        g_rp = np.ctypeslib.as_array(ctypes.cast(rp, ctypes.POINTER(ctypes.c_int64)), (nloc + 1,)).copy()
        if g:
            g_col = np.ctypeslib.as_array(ctypes.cast(gc, ctypes.POINTER(ctypes.c_int32)), (g,)).copy()
            g_w = np.ctypeslib.as_array(ctypes.cast(gw, ctypes.POINTER(ctypes.c_double)), (g,)).copy()
        else:
            g_col = np.empty(0, np.int32)
            g_w = np.empty(0, np.float64)
    finally:
        L.orc_free(rp)
        L.orc_free(gc)
        L.orc_free(gw)
    return g_rp, g_col, g_w, diag, nnzc


def build(row_ptr, col_idx, val, ncols=None, scale_rows=1, drop_tol=0.0, row_begin=0, row_end=None,
          keep_intermediates=False, threads=1):
    """Full oracle pipeline: [scale] -> CSC -> Gustavson rows -> graph."""
    row_ptr, col_idx, val = _c(row_ptr, np.int64), _c(col_idx, np.int32), _c(val, np.float64)
    nrows = row_ptr.size - 1
    ncols = nrows if ncols is None else int(ncols)
    a_hat = scale(row_ptr, val)[0] if scale_rows else val
    csc = transpose(nrows, ncols, row_ptr, col_idx, a_hat)
    f, _ = row_products(row_ptr, col_idx, csc[0])
    row_end = nrows if row_end is None else row_end
    g_rp, g_col, g_w, diag, nnzc = build_from_scaled(nrows, ncols, row_ptr, col_idx, a_hat, csc, drop_tol,
                                                     row_begin, row_end, threads=threads)
    products = int(f[row_begin:row_end].sum())
    return Graph(g_rp, g_col, g_w, diag, nnzc, row_begin, products,
                 a_hat if keep_intermediates else None, csc if keep_intermediates else None)


def cutsize(g_row_ptr, g_col, g_w, part, K, row_begin=0):
    """Returns (cut, total, intra)."""
    g_row_ptr, g_col, g_w = _c(g_row_ptr, np.int64), _c(g_col, np.int32), _c(g_w, np.float64)
    part = _c(part, np.int32)
    out = (ctypes.c_double * 3)()
    st = lib().orc_cutsize(g_row_ptr.size - 1, row_begin, _p(g_row_ptr), _p(g_col), _p(g_w), part.size,
                           _p(part), int(K), ctypes.byref(out, 0), ctypes.byref(out, 8), ctypes.byref(out, 16))
    if st:
        raise OracleError(st, "cutsize")
    return out[0], out[1], out[2]


def ip_matrix(g_row_ptr, g_col, g_w, part, K, row_begin=0, a_row_ptr=None):
    """Inter-block inner-product matrix ip[K, K] and part
    weights W[K]: unit weights, or nnz(r_i)
    when A's row pointers are given.  Returns (ip, W)."""
    g_row_ptr, g_col, g_w = _c(g_row_ptr, np.int64), _c(g_col, np.int32), _c(g_w, np.float64)
    part = _c(part, np.int32)
    ip = np.zeros((K, K), dtype=np.float64)
    W = np.zeros(K, dtype=np.int64)
    arp = _c(a_row_ptr, np.int64) if a_row_ptr is not None else None
    st = lib().orc_ip_matrix(g_row_ptr.size - 1, row_begin, _p(g_row_ptr), _p(g_col), _p(g_w), part.size,
                             _p(part), int(K), _p(arp) if arp is not None else None, _p(ip), _p(W))
    if st:
        raise OracleError(st, "ip_matrix")
    return ip, W


def dense_threshold(n):
    """T = ceil(sqrt(n)) (reading R20)."""
    return int(lib().orc_dense_threshold(int(n)))


def sparsify(row_ptr, col_idx, val, ncols=None):
    """A~: columns with more than T nonzeros keep their T largest |values|,
    ties to the lower row.  Returns (row_ptr, col, val)."""
    row_ptr, col_idx, val = _c(row_ptr, np.int64), _c(col_idx, np.int32), _c(val, np.float64)
    nrows = row_ptr.size - 1
    ncols = nrows if ncols is None else int(ncols)
    nnz = int(row_ptr[-1])
    orp = np.empty(nrows + 1, dtype=np.int64)
    oc = np.empty(max(nnz, 1), dtype=np.int32)
    ov = np.empty(max(nnz, 1), dtype=np.float64)
    nout = ctypes.c_int64()
    st = lib().orc_sparsify(nrows, ncols, _p(row_ptr), _p(col_idx), _p(val), _p(orp), _p(oc), _p(ov),
                            ctypes.byref(nout))
    if st:
        raise OracleError(st, "sparsify")
    return orp, oc[:nout.value].copy(), ov[:nout.value].copy()


def int_weights(w, alpha):
    """wgt = ceil(alpha * w), exact."""
    w = _c(w, np.float64)
    out = np.empty(w.size, dtype=np.int64)
    st = lib().orc_int_weights(w.size, _p(w), int(alpha), _p(out))
    if st:
        raise OracleError(st, "int_weights")
    return out
