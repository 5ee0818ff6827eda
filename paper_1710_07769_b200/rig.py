"""Thin ctypes binding over librig.so (include/rig.h).  Argument marshalling
only: every step of the path runs in the library's CUDA kernels.  PyTorch
supplies device memory and the current stream.  There is no CPU fallback: if
librig.so is missing the import of this module fails loudly.
"""
from __future__ import annotations

import ctypes
import os
import re

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RIG_LIB_VARIANT") or os.path.join(_HERE, "librig.so")
HEADER = os.path.join(os.path.dirname(_HERE), "include", "rig.h")

RIG_OK = 0
RIG_ERR_INVALID = -1
RIG_ERR_NONCANONICAL = -2
RIG_ERR_ZERO_ROW = -3
RIG_ERR_NONFINITE = -4
RIG_ERR_NOMEM = -5
RIG_ERR_CUDA = -6
RIG_FLAG_VALIDATE = 0x1
RIG_FLAG_DIAG = 0x2
RIG_FLAG_SPARSIFY = 0x4


class rig_csr_t(ctypes.Structure):
    _fields_ = [("nrows", ctypes.c_int64), ("ncols", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("row_ptr", ctypes.c_void_p), ("col_idx", ctypes.c_void_p), ("val", ctypes.c_void_p)]


class rig_graph_t(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("nnz", ctypes.c_int64), ("row_ptr", ctypes.c_void_p),
                ("col_idx", ctypes.c_void_p), ("w", ctypes.c_void_p), ("diag", ctypes.c_void_p)]


class RigError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"librig error {code}: {msg}")
        self.code = code


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"librig.so not built ({LIB_PATH}); run `python -m paper_1710_07769_b200.build` "
                          "or __graft_entry__.build() -- there is no CPU fallback")
    L = ctypes.CDLL(LIB_PATH)
    P, I64, I32, U32, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32, ctypes.c_double
    L.rig_build.argtypes = [P, ctypes.c_int, D, U32, P, P]
    L.rig_build_rows.argtypes = [P, ctypes.c_int, D, U32, I64, I64, P, P]
    L.rig_build_cut.argtypes = [P, ctypes.c_int, D, U32, I64, I64, P, I32, P, P, P]
    L.rig_graph_free.argtypes = [P, P]
    L.rig_plan_create.argtypes = [P, ctypes.c_int, D, U32, I64, I64, P, P]
    L.rig_plan_query.argtypes = [P, P, P, P]
    L.rig_plan_execute.argtypes = [P, P, P, P]
    L.rig_plan_destroy.argtypes = [P]
    L.rig_row_split.argtypes = [P, I32, P, P]
    L.rig_cutsize.argtypes = [P, I64, I64, P, I32, P, P]
    L.rig_build_host.argtypes = [P, ctypes.c_int, D, U32, P, I32, P, I64, P, P]
    L.rig_partition_ip.argtypes = [P, I64, I64, P, I32, P, P, P, P]
    L.rig_partition_ip_finalize.argtypes = [P, I32, P]
    L.rig_sparsify.argtypes = [P, ctypes.c_int, U32, P, P]
    L.rig_csr_free.argtypes = [P, P]
    L.rig_int_weights.argtypes = [P, I64, I64, P, P]
    L.rig_hem_match.argtypes = [P, P, P, I64, I32, P, P]
    L.rig_coarsen.argtypes = [P, P, P, P, I64, P, P, P]
    L.rig_coarse_free.argtypes = [P, P]
    L.rig_last_error.restype = ctypes.c_char_p
    L.rig_launch_count.restype = ctypes.c_uint64
    L.rig_version.restype = ctypes.c_char_p
    L.rig_last_path.restype = ctypes.c_char_p
    L.rig_profile_enable.argtypes = [ctypes.c_int]
    L.rig_profile_read.argtypes = [P, P]
    L.rig_pass_name.argtypes = [ctypes.c_int]
    L.rig_pass_name.restype = ctypes.c_char_p
    return L


lib = _load()


def header_symbols(path=HEADER):
    """Names of the functions include/rig.h declares."""
    with open(path) as fh:
        return re.findall(r"^RIG_API\s+[\w\s\*]+?\b(rig_\w+)\s*\(", fh.read(), flags=re.M)


def _check(code):
    if code != RIG_OK:
        raise RigError(code, lib.rig_last_error().decode())


def _stream(stream=None):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def rig_mem_stats(reset=False):
    """(bytes in use, high-water mark) of the device's stream-ordered pool,
    which holds every library allocation."""
    now, high = ctypes.c_uint64(), ctypes.c_uint64()
    _check(lib.rig_mem_stats(ctypes.byref(now), ctypes.byref(high), int(bool(reset))))
    return now.value, high.value


def rig_gather_probe(A: CSR, scale_rows=1, stream=None) -> float:
    """Measurement: the numeric pass's gather loop alone (k_gather_probe)."""
    out = ctypes.c_double()
    _check(lib.rig_gather_probe(ctypes.byref(A.c()), int(scale_rows), ctypes.byref(out), _stream(stream)))
    return out.value


def last_path() -> str:
    """Numeric path of this thread's last build: merge / rowwin / mixed."""
    return lib.rig_last_path().decode()


def launch_count() -> int:
    return int(lib.rig_launch_count())


class CSR:
    """Device CSR: row_ptr int64[n+1], col_idx int32[nnz], val float64[nnz]."""

    def __init__(self, row_ptr, col_idx, val, ncols=None, device="cuda"):
        self.row_ptr = torch.as_tensor(row_ptr, dtype=torch.int64, device=device).contiguous()
        self.col_idx = torch.as_tensor(col_idx, dtype=torch.int32, device=device).contiguous()
        self.val = torch.as_tensor(val, dtype=torch.float64, device=device).contiguous()
        self.nrows = self.row_ptr.numel() - 1
        self.ncols = self.nrows if ncols is None else int(ncols)
        self.nnz = self.col_idx.numel()

    def c(self):
        return rig_csr_t(self.nrows, self.ncols, self.nnz, self.row_ptr.data_ptr(), self.col_idx.data_ptr(),
                         self.val.data_ptr())


class _Cai:
    """__cuda_array_interface__ view over library-owned device memory."""

    def __init__(self, ptr, n, typestr, owner):
        self.owner = owner
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": typestr, "data": (int(ptr or 0), False),
                                         "version": 3, "strides": None, "stream": None}


class _GraphOwner:
    """Owns the library-allocated arrays of one graph; freed (rig_graph_free)
    when the Graph and every tensor view of it are gone.  The free is ordered
    on the stream and device the graph was BUILT on (not whatever is current at
    collection time), so it follows the build's pending work; a consumer on
    another stream must synchronise with the build stream before dropping its
    views.  Holds no reference back to the views: no reference cycle."""

    def __init__(self, g: rig_graph_t, stream=None):
        self.g = g
        s = stream if stream is not None else torch.cuda.current_stream()
        self.stream = s if isinstance(s, torch.cuda.Stream) else None
        self.raw_stream = _stream(stream)
        self.device = torch.cuda.current_device()

    def __del__(self):
        try:
            if self.g is not None:
                with torch.cuda.device(self.device):
                    lib.rig_graph_free(ctypes.byref(self.g), self.raw_stream)
                self.g = None
        except Exception:
            pass


class Graph:
    """G_RIP rows [row_begin, row_begin+n): library-owned device arrays
    (rig_build) exposed as torch views, created on first access."""

    def __init__(self, g: rig_graph_t, row_begin: int, stream):
        self._owner = _GraphOwner(g, stream)
        self._g = rig_graph_t(g.n, g.nnz, g.row_ptr, g.col_idx, g.w, g.diag)
        self.row_begin = row_begin
        self.n, self.nnz = int(g.n), int(g.nnz)
        self._views = {}

    def _view(self, name, ptr, n, typestr, dt):
        v = self._views.get(name)
        if v is None:
            dev = torch.device("cuda", torch.cuda.current_device())
            v = (torch.as_tensor(_Cai(ptr, n, typestr, self._owner), device=dev) if n
                 else torch.empty(0, dtype=dt, device=dev))
            self._views[name] = v
        return v

    @property
    def row_ptr(self):
        return self._view("row_ptr", self._g.row_ptr, self.n + 1, "<i8", torch.int64)

    @property
    def col_idx(self):
        return self._view("col_idx", self._g.col_idx, self.nnz, "<i4", torch.int32)

    @property
    def w(self):
        return self._view("w", self._g.w, self.nnz, "<f8", torch.float64)

    @property
    def diag(self):
        return self._view("diag", self._g.diag, self.n, "<f8", torch.float64) if self._g.diag else None

    def c(self):
        return self._g


class TensorGraph:
    """Graph in torch-owned arrays (staged API)."""

    def __init__(self, row_ptr, col_idx, w, diag, row_begin):
        self.row_ptr, self.col_idx, self.w, self.diag = row_ptr, col_idx, w, diag
        self.row_begin = row_begin
        self.n = row_ptr.numel() - 1
        self.nnz = col_idx.numel()

    def c(self):
        return rig_graph_t(self.n, self.nnz, self.row_ptr.data_ptr(), self.col_idx.data_ptr(), self.w.data_ptr(),
                           self.diag.data_ptr() if self.diag is not None else None)


def rig_build(A: CSR, scale_rows=1, drop_tol=0.0, flags=0, stream=None) -> Graph:
    g = rig_graph_t()
    s = _stream(stream)
    _check(lib.rig_build(ctypes.byref(A.c()), int(scale_rows), float(drop_tol), int(flags), ctypes.byref(g), s))
    return Graph(g, 0, stream)


def rig_build_rows(A: CSR, row_begin, row_end, scale_rows=1, drop_tol=0.0, flags=0, stream=None) -> Graph:
    g = rig_graph_t()
    s = _stream(stream)
    _check(lib.rig_build_rows(ctypes.byref(A.c()), int(scale_rows), float(drop_tol), int(flags), int(row_begin),
                              int(row_end), ctypes.byref(g), s))
    return Graph(g, int(row_begin), stream)


def rig_build_cut(A: CSR, part: torch.Tensor, K: int, row_begin=0, row_end=None, scale_rows=1, drop_tol=0.0,
                  flags=0, out=None, stream=None):
    """Whole hot path in one call: graph rows [row_begin, row_end) and the
    cutsize of `part` over them (device float64[1], asynchronous value)."""
    g = rig_graph_t()
    row_end = A.nrows if row_end is None else int(row_end)
    if out is None:
        out = torch.empty(1, dtype=torch.float64, device=part.device)
    _check(lib.rig_build_cut(ctypes.byref(A.c()), int(scale_rows), float(drop_tol), int(flags), int(row_begin),
                             row_end, ctypes.c_void_p(part.data_ptr()), int(K), ctypes.byref(g),
                             ctypes.c_void_p(out.data_ptr()), _stream(stream)))
    return Graph(g, int(row_begin), stream), out


class Plan:
    """Staged API: rig_plan_create (a0-a4) -> query -> execute (a5-a6)."""

    def __init__(self, A: CSR, scale_rows=1, drop_tol=0.0, flags=0, row_begin=0, row_end=None, stream=None):
        self.A = A  # keep inputs alive
        self.row_begin = int(row_begin)
        self.row_end = A.nrows if row_end is None else int(row_end)
        self.flags = int(flags)
        self._p = ctypes.c_void_p()
        _check(lib.rig_plan_create(ctypes.byref(A.c()), int(scale_rows), float(drop_tol), self.flags,
                                   self.row_begin, self.row_end, ctypes.byref(self._p), _stream(stream)))
        nu, pr, ws = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_size_t()
        _check(lib.rig_plan_query(self._p, ctypes.byref(nu), ctypes.byref(pr), ctypes.byref(ws)))
        self.nnz_upper, self.products, self.workspace_bytes = nu.value, pr.value, ws.value

    def execute(self, stream=None) -> TensorGraph:
        n = self.row_end - self.row_begin
        dev = self.A.row_ptr.device
        rp = torch.empty(n + 1, dtype=torch.int64, device=dev)
        col = torch.empty(max(self.nnz_upper, 1), dtype=torch.int32, device=dev)
        w = torch.empty(max(self.nnz_upper, 1), dtype=torch.float64, device=dev)
        diag = torch.empty(max(n, 1), dtype=torch.float64, device=dev) if self.flags & RIG_FLAG_DIAG else None
        ws = torch.empty(max(self.workspace_bytes, 1), dtype=torch.uint8, device=dev)
        g = rig_graph_t(n, self.nnz_upper, rp.data_ptr(), col.data_ptr(), w.data_ptr(),
                        diag.data_ptr() if diag is not None else None)
        _check(lib.rig_plan_execute(self._p, ctypes.c_void_p(ws.data_ptr()), ctypes.byref(g), _stream(stream)))
        return TensorGraph(rp, col[:g.nnz], w[:g.nnz], diag[:n] if diag is not None else None, self.row_begin)

    def destroy(self):
        if self._p:
            lib.rig_plan_destroy(self._p)
            self._p = ctypes.c_void_p()

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


def rig_row_split(A: CSR, parts: int, stream=None):
    split = (ctypes.c_int64 * (parts + 1))()
    _check(lib.rig_row_split(ctypes.byref(A.c()), int(parts), split, _stream(stream)))
    return [int(x) for x in split]


def rig_cutsize(g, part: torch.Tensor, K: int, n_global=None, out=None, stream=None) -> torch.Tensor:
    """Asynchronous: returns a device float64[1] tensor."""
    part = part if part.dtype == torch.int32 else part.to(torch.int32)
    n_global = part.numel() if n_global is None else int(n_global)
    if out is None:
        out = torch.empty(1, dtype=torch.float64, device=part.device)
    gc = g.c()
    _check(lib.rig_cutsize(ctypes.byref(gc), int(g.row_begin), n_global, ctypes.c_void_p(part.data_ptr()), int(K),
                           ctypes.c_void_p(out.data_ptr()), _stream(stream)))
    return out


def rig_partition_ip_accumulate(g, part: torch.Tensor, K: int, a_row_ptr=None, acc=None, W=None, n_global=None,
                                stream=None):
    """Accumulate the fixed-point inter-block inner products and part weights
    of graph (shard) g into device int64 tensors acc [4K^2+1] and W [K]
    (zeroed here when not given).  Asynchronous.  Multi-GPU: all_reduce(SUM)
    both, then rig_partition_ip_finalize."""
    part = part if part.dtype == torch.int32 else part.to(torch.int32)
    n_global = part.numel() if n_global is None else int(n_global)
    dev = part.device
    if acc is None:
        acc = torch.zeros(4 * K * K + 1, dtype=torch.int64, device=dev)
    if W is None:
        W = torch.zeros(K, dtype=torch.int64, device=dev)
    gc = g.c()
    arp = ctypes.c_void_p(a_row_ptr.data_ptr()) if a_row_ptr is not None else None
    _check(lib.rig_partition_ip(ctypes.byref(gc), int(g.row_begin), n_global, ctypes.c_void_p(part.data_ptr()), int(K),
                                arp, ctypes.c_void_p(acc.data_ptr()), ctypes.c_void_p(W.data_ptr()), _stream(stream)))
    return acc, W


def rig_partition_ip_finalize(acc, K: int):
    """Host conversion of the accumulated limbs: returns a float64 [K, K]
    CPU tensor (ip_km)."""
    a = acc.detach().to("cpu", torch.int64).contiguous()
    ip = torch.empty((K, K), dtype=torch.float64)
    _check(lib.rig_partition_ip_finalize(ctypes.c_void_p(a.data_ptr()), int(K), ctypes.c_void_p(ip.data_ptr())))
    return ip


def rig_partition_ip(g, part: torch.Tensor, K: int, a_row_ptr=None, stream=None):
    """ip [K, K] (CPU float64) and part weights W [K] (CPU int64) of graph g
    under `part`.  Synchronises (reads the result)."""
    acc, W = rig_partition_ip_accumulate(g, part, K, a_row_ptr, stream=stream)
    return rig_partition_ip_finalize(acc, K), W.cpu()


def rig_sparsify(A: CSR, scale_rows=1, flags=0, stream=None) -> CSR:
    """A~ as a torch-owned device CSR
    (the library's arrays are copied, then released).  Synchronises."""
    out = rig_csr_t()
    _check(lib.rig_sparsify(ctypes.byref(A.c()), int(scale_rows), int(flags), ctypes.byref(out), _stream(stream)))
    try:
        dev = torch.device("cuda", torch.cuda.current_device())

        def view(ptr, n, ts, dt):
            return (torch.as_tensor(_Cai(ptr, n, ts, None), device=dev).clone() if n
                    else torch.empty(0, dtype=dt, device=dev))

        rp = view(out.row_ptr, out.nrows + 1, "<i8", torch.int64)
        ci = view(out.col_idx, out.nnz, "<i4", torch.int32)
        v = view(out.val, out.nnz, "<f8", torch.float64)
    finally:
        lib.rig_csr_free(ctypes.byref(out), _stream(stream))
    return CSR(rp, ci, v, ncols=out.ncols if out.ncols else A.ncols, device=dev)


def rig_int_weights(w: torch.Tensor, alpha: int, out=None, stream=None) -> torch.Tensor:
    """wgt = ceil(alpha * w) exactly, device int64; -1 marks
    an invalid element.  Asynchronous."""
    w = w.contiguous()
    if out is None:
        out = torch.empty(w.numel(), dtype=torch.int64, device=w.device)
    _check(lib.rig_int_weights(ctypes.c_void_p(w.data_ptr()), int(w.numel()), int(alpha),
                               ctypes.c_void_p(out.data_ptr()), _stream(stream)))
    return out


class rig_coarse_t(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("nnz", ctypes.c_int64), ("row_ptr", ctypes.c_void_p),
                ("col_idx", ctypes.c_void_p), ("wgt", ctypes.c_void_p), ("vwgt", ctypes.c_void_p),
                ("cmap", ctypes.c_void_p)]


def rig_hem_match(row_ptr: torch.Tensor, col: torch.Tensor, wgt: torch.Tensor, rounds=4, stream=None) -> torch.Tensor:
    """f4 (R23): heavy-edge matching of a symmetric device graph
    with int64 edge weights; returns match (device int32, partner or -1)."""
    n = row_ptr.numel() - 1
    match = torch.empty(max(n, 1), dtype=torch.int32, device=row_ptr.device)
    _check(lib.rig_hem_match(ctypes.c_void_p(row_ptr.data_ptr()), ctypes.c_void_p(col.data_ptr()),
                             ctypes.c_void_p(wgt.data_ptr()), n, int(rounds), ctypes.c_void_p(match.data_ptr()),
                             _stream(stream)))
    return match[:n]


def rig_coarsen(row_ptr, col, wgt, match, vwgt=None, stream=None):
    """f4 (R24-R25): one coarsening step.  Returns a dict of device
    tensors (row_ptr, col_idx, wgt, vwgt, cmap) and the coarse sizes; the
    library block is copied into torch tensors and released."""
    n = row_ptr.numel() - 1
    c = rig_coarse_t()
    vp = ctypes.c_void_p(vwgt.data_ptr()) if vwgt is not None else None
    _check(lib.rig_coarsen(ctypes.c_void_p(row_ptr.data_ptr()), ctypes.c_void_p(col.data_ptr()),
                           ctypes.c_void_p(wgt.data_ptr()), vp, n, ctypes.c_void_p(match.data_ptr()),
                           ctypes.byref(c), _stream(stream)))
    out = {"n": int(c.n), "nnz": int(c.nnz)}
    if c.row_ptr:
        for name, ptr, cnt, ts, dt in (("row_ptr", c.row_ptr, c.n + 1, "<i8", torch.int64),
                                       ("col_idx", c.col_idx, c.nnz, "<i4", torch.int32),
                                       ("wgt", c.wgt, c.nnz, "<i8", torch.int64),
                                       ("vwgt", c.vwgt, c.n, "<i8", torch.int64),
                                       ("cmap", c.cmap, n, "<i4", torch.int32)):
            out[name] = torch.as_tensor(_Cai(ptr, cnt, ts, None), device=row_ptr.device).clone() if cnt else \
                torch.empty(0, dtype=dt, device=row_ptr.device)
        _check(lib.rig_coarse_free(ctypes.byref(c), _stream(stream)))
    return out


def rig_build_host(row_ptr, col_idx, val, ncols, scale_rows, drop_tol, flags, part, K, out_row_ptr, out_col,
                   out_w, out_diag=None, stream=None):
    """End-to-end from HOST (ideally pinned) torch CPU tensors.  Returns
    (nnz, cut).  Output tensors are caller-allocated host arrays."""
    n = row_ptr.numel() - 1
    A = rig_csr_t(n, int(ncols), col_idx.numel(), row_ptr.data_ptr(), col_idx.data_ptr(), val.data_ptr())
    g = rig_graph_t(n, 0, out_row_ptr.data_ptr(), out_col.data_ptr(), out_w.data_ptr(),
                    out_diag.data_ptr() if out_diag is not None else None)
    cut = ctypes.c_double()
    code = lib.rig_build_host(ctypes.byref(A), int(scale_rows), float(drop_tol), int(flags),
                              ctypes.c_void_p(part.data_ptr()) if part is not None else None, int(K), ctypes.byref(g),
                              int(out_col.numel()), ctypes.byref(cut), _stream(stream))
    if code != RIG_OK:
        raise RigError(code, lib.rig_last_error().decode() + f" (required capacity {g.nnz})")
    return int(g.nnz), cut.value
