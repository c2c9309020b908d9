"""Thin ctypes binding of librg (include/rg.h): argument marshalling only.

Every function here has the name of the C entry point it wraps and does nothing but convert
numpy arrays / torch tensors to pointers, call the library and raise on a non-OK status.  All
arithmetic runs in the CUDA kernels of ``csrc/``; there is no CPU fallback: if ``lib/librg.so`` is
missing, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RG_LIB_PATH") or os.path.join(_HERE, "lib", "librg.so")  # override: A/B experiments

RG_OK, RG_E_INVAL, RG_E_NOMEM, RG_E_CUDA, RG_E_STATE, RG_E_SINGULAR, RG_E_NUMERIC, RG_E_CHECK = range(8)
RG_CSR, RG_BSR = 0, 1
RG_PLAIN, RG_AUGMENT, RG_DEFLATE, RG_OBLIQUE, RG_ORTHOGONAL = 0, 1, 2, 3, 4
RG_HOST, RG_DEVICE = 0, 1
RG_FLAG_NO_GRAPH, RG_FLAG_PROFILE, RG_FLAG_CGS2, RG_FLAG_NO_PERSIST, RG_FLAG_KEEP_BASIS = 1, 2, 4, 8, 16
RG_EXPORT_W, RG_EXPORT_Q, RG_EXPORT_RC, RG_EXPORT_V, RG_EXPORT_H, RG_EXPORT_B = 0, 1, 2, 3, 4, 5
RG_MODES_LARGEST, RG_MODES_SMALLEST = 0, 1
RG_PREC_NONE, RG_PREC_SSOR = 0, 1
PRECS = {None: RG_PREC_NONE, "none": RG_PREC_NONE, "ssor": RG_PREC_SSOR}
MODES = {"largest": RG_MODES_LARGEST, "smallest": RG_MODES_SMALLEST}
VARIANTS = {"plain": RG_PLAIN, "augment": RG_AUGMENT, "deflate": RG_DEFLATE, "oblique": RG_OBLIQUE,
            "orthogonal": RG_ORTHOGONAL}
STATUS = {0: "RG_OK", 1: "RG_E_INVAL", 2: "RG_E_NOMEM", 3: "RG_E_CUDA", 4: "RG_E_STATE",
          5: "RG_E_SINGULAR", 6: "RG_E_NUMERIC", 7: "RG_E_CHECK"}

# Symbols declared in include/rg.h (tests check the .so exports exactly these).
SYMBOLS = ("rg_create", "rg_update_matrix", "rg_matrix_values", "rg_push_snapshot", "rg_clear_snapshots", "rg_build_recycle", "rg_build_recycle_modes",
           "rg_solve", "rg_apply", "rg_set_preconditioner", "rg_apply_preconditioner", "rg_export",
           "rg_kernel_stats", "rg_kernel_trace", "rg_reset_kernel_stats", "rg_destroy", "rg_last_error")


class RgError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class rg_matrix(ctypes.Structure):
    _fields_ = [("fmt", ctypes.c_int), ("n_rows", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("block", ctypes.c_int32), ("row_ptr", ctypes.c_void_p), ("col_idx", ctypes.c_void_p),
                ("val", ctypes.c_void_p), ("mem", ctypes.c_int), ("sell_C", ctypes.c_int32),
                ("sell_sigma", ctypes.c_int32)]


class rg_options(ctypes.Structure):
    _fields_ = [("max_m", ctypes.c_int32), ("max_snapshots", ctypes.c_int32), ("max_k", ctypes.c_int32),
                ("cuda_stream", ctypes.c_void_p), ("flags", ctypes.c_int32)]


class rg_report(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int32), ("restarts", ctypes.c_int32), ("converged", ctypes.c_int32),
                ("k_eff", ctypes.c_int32), ("spmv_count", ctypes.c_int32), ("history_len", ctypes.c_int32),
                ("rel_residual", ctypes.c_double), ("ms_total", ctypes.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class rg_kstat(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 24), ("launches", ctypes.c_int64), ("noop_launches", ctypes.c_int64),
                ("total_ms", ctypes.c_double), ("tail_ms", ctypes.c_double), ("bytes", ctypes.c_double)]


class rg_trace_event(ctypes.Structure):
    _fields_ = [("t_ns", ctypes.c_int64), ("kind", ctypes.c_int32), ("name", ctypes.c_char * 20)]


def load(path: str = LIB_PATH):
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: build it with __graft_entry__.build() (no CPU fallback exists)")
    L = ctypes.CDLL(path)
    vp, i32, i64, d = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    L.rg_create.argtypes = [ctypes.POINTER(vp), i64, ctypes.POINTER(rg_matrix), ctypes.POINTER(rg_options)]
    L.rg_update_matrix.argtypes = [vp, ctypes.POINTER(rg_matrix)]
    L.rg_matrix_values.argtypes = [vp, ctypes.POINTER(vp), ctypes.POINTER(i64)]
    L.rg_push_snapshot.argtypes = [vp, vp, ctypes.c_int]
    L.rg_clear_snapshots.argtypes = [vp]
    L.rg_build_recycle.argtypes = [vp, i32, ctypes.POINTER(i32), vp]
    L.rg_build_recycle_modes.argtypes = [vp, i32, i32, ctypes.POINTER(i32), vp]
    L.rg_solve.argtypes = [vp, vp, vp, i32, ctypes.c_int, d, i32, vp, ctypes.c_int, vp, i32,
                           ctypes.POINTER(rg_report)]
    L.rg_apply.argtypes = [vp, vp, vp, ctypes.c_int]
    L.rg_set_preconditioner.argtypes = [vp, i32, d, vp, ctypes.c_int, ctypes.POINTER(i32)]
    L.rg_apply_preconditioner.argtypes = [vp, vp, vp, ctypes.c_int]
    L.rg_export.argtypes = [vp, i32, vp, ctypes.c_int, ctypes.POINTER(i32)]
    L.rg_kernel_stats.argtypes = [vp, ctypes.POINTER(rg_kstat), i32, ctypes.POINTER(i32)]
    L.rg_kernel_trace.argtypes = [vp, ctypes.POINTER(rg_trace_event), i32, ctypes.POINTER(i32)]
    L.rg_reset_kernel_stats.argtypes = [vp]
    L.rg_destroy.argtypes = [vp]
    L.rg_destroy.restype = None
    L.rg_last_error.restype = ctypes.c_char_p
    for f in SYMBOLS:
        if f not in ("rg_destroy", "rg_last_error"):
            getattr(L, f).restype = ctypes.c_int
    return L


_lib = load()


def _check(st):
    if st != RG_OK:
        raise RgError(st, _lib.rg_last_error().decode())


_CTX_N = {}  # context handle -> n (argument checks only)

_DT_NAMES = {np.float64: ("float64", "torch.float64"), np.int32: ("int32", "torch.int32")}


def _ptr(a, dtype=np.float64, min_len=None, name="array"):
    """(pointer, mem) of a numpy array or torch tensor (None -> (None, None)).

    Checks what the C ABI cannot: element type (float64 values, int32 indices), contiguity and,
    when min_len is given, that at least min_len elements are there (the library reads or writes
    that many through the raw pointer)."""
    if a is None:
        return None, None
    np_name, torch_name = _DT_NAMES[dtype]
    if isinstance(a, np.ndarray):
        if a.dtype != np.dtype(dtype):
            raise TypeError(f"{name}: dtype {a.dtype}, expected {np_name}")
        if not a.flags.c_contiguous:
            raise ValueError(f"{name}: arrays must be contiguous")
        if min_len is not None and a.size < min_len:
            raise ValueError(f"{name}: {a.size} elements, at least {min_len} needed")
        return a.ctypes.data, RG_HOST
    # torch tensor
    if str(a.dtype) != torch_name:
        raise TypeError(f"{name}: dtype {a.dtype}, expected {torch_name}")
    if not a.is_contiguous():
        raise ValueError(f"{name}: tensors must be contiguous")
    if min_len is not None and a.numel() < min_len:
        raise ValueError(f"{name}: {a.numel()} elements, at least {min_len} needed")
    return a.data_ptr(), (RG_DEVICE if a.is_cuda else RG_HOST)


def _n(ctx):
    return _CTX_N.get(ctx.value if hasattr(ctx, "value") else ctx)


def _mem(a):
    if isinstance(a, np.ndarray):
        return RG_HOST
    return RG_DEVICE if a.is_cuda else RG_HOST


def _mem_of(*arrays):
    mems = {_mem(a) for a in arrays if a is not None}
    if len(mems) > 1:
        raise ValueError("all arrays of one call must live in the same memory (host or device)")
    return mems.pop() if mems else RG_HOST


def make_matrix(n, row_ptr, col_idx, val, fmt="csr", block=1, sell_C=0, keep=None, sell_sigma=1):
    """Build an rg_matrix descriptor.  row_ptr/col_idx None -> values-only update.  Arrays must
    stay alive during the call (`keep` collects references)."""
    arrs = [a for a in (row_ptr, col_idx, val) if a is not None]
    mem = _mem_of(*arrs)
    if keep is not None:
        keep.extend(arrs)
    if fmt == "bsr":
        nnz = int(col_idx.shape[0]) if col_idx is not None else int(val.shape[0]) // (block * block)
        nrows, vlen = int(n) // int(block), nnz * int(block) * int(block)
    else:
        nnz = int(val.shape[0])
        nrows, vlen = int(n), nnz
    rp, _ = _ptr(row_ptr, np.int32, nrows + 1, "row_ptr")
    ci, _ = _ptr(col_idx, np.int32, nnz, "col_idx")
    v, _ = _ptr(val, np.float64, vlen, "val")
    return rg_matrix(RG_BSR if fmt == "bsr" else RG_CSR, int(n), nnz, int(block), rp, ci, v, mem, int(sell_C),
                     int(sell_sigma))


def rg_create(n, A: rg_matrix, max_m=64, max_snapshots=32, max_k=32, stream=None, flags=0):
    ctx = ctypes.c_void_p()
    opt = rg_options(int(max_m), int(max_snapshots), int(max_k), stream, int(flags))
    _check(_lib.rg_create(ctypes.byref(ctx), int(n), ctypes.byref(A), ctypes.byref(opt)))
    _CTX_N[ctx.value] = int(n)
    return ctx


def rg_update_matrix(ctx, A: rg_matrix):
    _check(_lib.rg_update_matrix(ctx, ctypes.byref(A)))


def rg_matrix_values(ctx):
    """(device pointer, length) of the library-owned matrix values."""
    p = ctypes.c_void_p()
    n = ctypes.c_int64(0)
    _check(_lib.rg_matrix_values(ctx, ctypes.byref(p), ctypes.byref(n)))
    return p.value, n.value


def rg_update_values_inplace(ctx, n, nnz, fmt="csr", block=1, sell_C=0, sell_sigma=1):
    """rg_update_matrix with val == rg_matrix_values() (values already written in place)."""
    ptr, _ = rg_matrix_values(ctx)
    A = rg_matrix(RG_BSR if fmt == "bsr" else RG_CSR, int(n), int(nnz), int(block), None, None, ptr, RG_DEVICE,
                  int(sell_C), int(sell_sigma))
    _check(_lib.rg_update_matrix(ctx, ctypes.byref(A)))


def rg_push_snapshot(ctx, x):
    p, mem = _ptr(x, np.float64, _n(ctx), "x")
    _check(_lib.rg_push_snapshot(ctx, p, mem))


def rg_clear_snapshots(ctx):
    _check(_lib.rg_clear_snapshots(ctx))


def rg_build_recycle(ctx, k, n_snapshots=64, deferred=False):
    """deferred=True: asynchronous build (k_eff, sigma NULL), returns (None, None)."""
    if deferred:
        _check(_lib.rg_build_recycle(ctx, int(k), None, None))
        return None, None
    ke = ctypes.c_int32(0)
    sig = np.zeros(n_snapshots)
    _check(_lib.rg_build_recycle(ctx, int(k), ctypes.byref(ke), sig.ctypes.data))
    return ke.value, sig


def rg_build_recycle_modes(ctx, k, modes="largest", n_snapshots=64):
    ke = ctypes.c_int32(0)
    sig = np.zeros(n_snapshots)
    md = MODES[modes] if isinstance(modes, str) else int(modes)
    _check(_lib.rg_build_recycle_modes(ctx, int(k), md, ctypes.byref(ke), sig.ctypes.data))
    return ke.value, sig


def rg_solve(ctx, b, x_out, x0=None, m=30, variant="plain", tol=1e-8, max_iters=20000, history_cap=0):
    v = VARIANTS[variant] if isinstance(variant, str) else int(variant)
    mem = _mem_of(b, x_out, x0)
    n = _n(ctx)
    pb, _ = _ptr(b, np.float64, n, "b")
    px, _ = _ptr(x_out, np.float64, n, "x_out")
    p0, _ = _ptr(x0, np.float64, n, "x0")
    hist = np.zeros(max(history_cap, 1))
    rep = rg_report()
    _check(_lib.rg_solve(ctx, pb, p0, int(m), v, float(tol), int(max_iters), px, mem,
                         hist.ctypes.data if history_cap > 0 else None, int(history_cap), ctypes.byref(rep)))
    out = rep.as_dict()
    out["history"] = hist[: rep.history_len].copy()
    return out


def rg_apply(ctx, x, y):
    mem = _mem_of(x, y)
    n = _n(ctx)
    _check(_lib.rg_apply(ctx, _ptr(x, np.float64, n, "x")[0], _ptr(y, np.float64, n, "y")[0], mem))


def rg_set_preconditioner(ctx, kind="ssor", omega=1.0, colors=None):
    """colors: None (library greedy colouring) or an int32 array / tensor of length n."""
    kd = PRECS[kind] if (kind is None or isinstance(kind, str)) else int(kind)
    nc = ctypes.c_int32(0)
    p, mem = _ptr(colors, np.int32, _n(ctx), "colors")
    _check(_lib.rg_set_preconditioner(ctx, kd, float(omega), p, RG_HOST if mem is None else mem, ctypes.byref(nc)))
    return nc.value


def rg_apply_preconditioner(ctx, x, y):
    mem = _mem_of(x, y)
    n = _n(ctx)
    _check(_lib.rg_apply_preconditioner(ctx, _ptr(x, np.float64, n, "x")[0], _ptr(y, np.float64, n, "y")[0], mem))


def rg_export(ctx, which, out):
    """Copy an internal item into `out` (None: only return the count: k_eff for W / Q / R_C, the
    number of Arnoldi steps J for V / H / B).  The caller sizes `out` (include/rg.h)."""
    ke = ctypes.c_int32(0)
    p, mem = _ptr(out, np.float64, None, "out")
    _check(_lib.rg_export(ctx, int(which), p, RG_HOST if mem is None else mem, ctypes.byref(ke)))
    return ke.value


def rg_kernel_stats(ctx):
    buf = (rg_kstat * 64)()
    cnt = ctypes.c_int32(0)
    _check(_lib.rg_kernel_stats(ctx, buf, 64, ctypes.byref(cnt)))
    return {buf[i].name.decode(): dict(launches=buf[i].launches, noop=buf[i].noop_launches,
                                       ms=buf[i].total_ms, tail_ms=buf[i].tail_ms, bytes=buf[i].bytes)
            for i in range(cnt.value)}


def rg_kernel_trace(ctx, cap=65536):
    """Device kernel timeline since the last reset: list of (t_ns, kind, name), kind 0 start / 1 end /
    2 no-op (contexts created with RG_FLAG_PROFILE); plus the number of events recorded."""
    buf = (rg_trace_event * cap)()
    cnt = ctypes.c_int32(0)
    _check(_lib.rg_kernel_trace(ctx, buf, cap, ctypes.byref(cnt)))
    n = min(cnt.value, cap)
    return [(buf[i].t_ns, buf[i].kind, buf[i].name.decode()) for i in range(n)], cnt.value


def rg_reset_kernel_stats(ctx):
    _check(_lib.rg_reset_kernel_stats(ctx))


def rg_destroy(ctx):
    _CTX_N.pop(ctx.value if hasattr(ctx, "value") else ctx, None)
    _lib.rg_destroy(ctx)


def rg_last_error():
    return _lib.rg_last_error().decode()
