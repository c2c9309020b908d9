"""Seeded synthetic inputs for the five BASELINE.json configs (input generators only).

This package builds the sequences of systems ``A_t x_t = b_t`` (PAPER.md:95-118,
eq. ``sequence_linear_systems``; "the sequence of matrices and right-hand sides depend on the
previous solution") that stand in for the paper's deal.II benchmark.  It holds
none of the method's arithmetic: the oracle (``oracle/``) and the CUDA library
(``paper_1807_09467_b200``) both consume its outputs, and neither is imported here.

The recipe (stencils, seeds, sequence scalars) is DESIGN.md §"Input recipe"; the per-row formulas
live in ``synth_common.h`` and are compiled both for the host (``libsynth.so``) and for the device
(``libsynth_cuda.so``) so that the two produce bit-identical values.
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None
_CULIB = None

_i32p = ctypes.POINTER(ctypes.c_int32)
_f64p = ctypes.POINTER(ctypes.c_double)


def _ptr(a, t=_f64p):
    if a is None:
        return None
    return a.ctypes.data_as(t)


def lib():
    """Host generator library (``synth/libsynth.so``)."""
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "libsynth.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run __graft_entry__.build() (or `make -C synth`)")
        L = ctypes.CDLL(path)
        L.sy_fill5.restype = ctypes.c_int64
        L.sy_fill5.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                               ctypes.c_double, ctypes.c_double, _f64p, _i32p, _i32p, _f64p]
        L.sy_fill9.restype = ctypes.c_int64
        L.sy_fill9.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                               ctypes.c_double, _i32p, _i32p, _f64p]
        L.sy_fill7.restype = ctypes.c_int64
        L.sy_fill7.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                               ctypes.c_double, ctypes.c_double, ctypes.c_double, _i32p, _i32p, _f64p]
        L.sy_c5_pattern.restype = ctypes.c_int64
        L.sy_c5_pattern.argtypes = [ctypes.c_int, _i32p, _i32p, ctypes.POINTER(ctypes.c_int8)]
        L.sy_c5_values.restype = None
        L.sy_c5_values.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.c_uint64,
                                   ctypes.POINTER(ctypes.c_int8), ctypes.c_double, ctypes.c_double, _f64p]
        L.sy_c5_perturb.restype = None
        L.sy_c5_perturb.argtypes = [ctypes.c_int64, ctypes.c_uint64, ctypes.c_int, _f64p]
        L.sy_normal_vec.restype = None
        L.sy_normal_vec.argtypes = [ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint64, _f64p]
        L.sy_rhs.restype = None
        L.sy_rhs.argtypes = [ctypes.c_int64, _f64p, ctypes.c_double, ctypes.c_double, _f64p]
        L.sy_bumps.restype = None
        L.sy_bumps.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                               ctypes.c_double, ctypes.c_double, ctypes.c_uint64, _f64p]
        _LIB = L
    return _LIB


def culib():
    """Device generator library (``synth/libsynth_cuda.so``)."""
    global _CULIB
    if _CULIB is None:
        path = os.path.join(_HERE, "libsynth_cuda.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run __graft_entry__.build()")
        L = ctypes.CDLL(path)
        vp = ctypes.c_void_p
        L.syd_fill5_values.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                       ctypes.c_double, ctypes.c_double, vp, vp, vp, vp]
        L.syd_fill7_values.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                       ctypes.c_double, ctypes.c_double, ctypes.c_double, vp, vp, vp]
        L.syd_rhs.argtypes = [ctypes.c_int64, vp, ctypes.c_double, ctypes.c_double, vp, vp]
        L.syd_c5_values.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.c_uint64, vp, ctypes.c_double,
                                    ctypes.c_double, vp, vp]
        L.syd_c5_perturb.argtypes = [ctypes.c_int64, ctypes.c_uint64, ctypes.c_int, vp, vp]
        L.syd_normal_vec.argtypes = [ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint64, vp, vp]
        for f in ("syd_fill5_values", "syd_fill7_values", "syd_rhs", "syd_c5_values", "syd_c5_perturb",
                  "syd_normal_vec"):
            getattr(L, f).restype = ctypes.c_int
        _CULIB = L
    return _CULIB


# ----------------------------------------------------------------------------------------------
# The five configs (BASELINE.json "configs"; readings in DESIGN.md / SURVEY.md §8c-A8..A20).
# ----------------------------------------------------------------------------------------------
@dataclass(frozen=True)
class Config:
    name: str
    cid: int
    kind: str                 # "5pt", "9pt", "7pt", "bsr"
    N: int                    # grid points per axis (bsr: elements per axis E)
    nu: float = 0.0
    dt: float = 1.0
    systems: int = 1
    m: int = 30               # GMRES restart
    k: int = 5                # recycle dimension
    s: int = 10               # snapshot-window capacity
    fmt: str = "csr"          # csr | sell | bsr
    forcing: float = 0.0      # f in b_t = u_{t-1}/dt + f
    bumps: tuple = (3, 0.1, 1.0, 1.0)   # (count, width, amp_lo, amp_hi)
    B: int = 64               # bsr block size
    tol: float = 1e-8
    variants: tuple = ("plain", "augment", "deflate")
    extra: dict = field(default_factory=dict)

    @property
    def seed(self) -> int:
        return 1000 + self.cid

    @property
    def dim(self) -> int:
        return 3 if self.kind in ("7pt", "bsr") else 2

    @property
    def n(self) -> int:
        if self.kind == "bsr":
            return self.N ** 3 * self.B
        return self.N ** self.dim

    def reduced(self, N: int, **kw) -> "Config":
        d = dict(self.__dict__)
        d["N"] = N
        d.update(kw)
        return Config(**d)


CONFIGS = {
    "C1": Config("C1", 1, "5pt", 32, nu=0.01, dt=0.05, systems=10, m=30, k=5, s=10, forcing=1.0,
                 bumps=(3, 0.1, 1.0, 1.0)),
    "C2": Config("C2", 2, "5pt", 512, nu=1e-3, dt=0.01, systems=50, m=50, k=10, s=20, forcing=0.0,
                 bumps=(5, 0.05, 0.5, 1.0)),
    "C3": Config("C3", 3, "9pt", 1024, nu=1e-4, dt=0.01, systems=40, m=30, k=16, s=32, fmt="sell",
                 forcing=0.0, bumps=(3, 0.1, 1.0, 1.0)),
    "C4": Config("C4", 4, "7pt", 128, nu=5e-3, dt=0.02, systems=30, m=40, k=16, s=32, forcing=1.0,
                 bumps=(3, 0.1, 1.0, 1.0)),
    "C5": Config("C5", 5, "bsr", 32, systems=20, m=30, k=20, s=40, fmt="bsr", B=64),
}


def nnz_closed_form(cfg: Config) -> int:
    """Closed-form stored entries (blocks for bsr) of the config's pattern."""
    N = cfg.N
    if cfg.kind == "5pt":
        return 5 * N * N - 4 * N
    if cfg.kind == "9pt":
        return 9 * N * N - 12 * N
    if cfg.kind == "7pt":
        return 7 * N ** 3 - 6 * N ** 2
    if cfg.kind == "bsr":
        return N ** 3 + 6 * N * N * (N - 1)
    raise ValueError(cfg.kind)


def velocity(cfg: Config, t: int):
    """Constant-in-space velocity of system t (C1 rotating, C4 pulsating); None otherwise."""
    if cfg.name == "C1" or (cfg.kind == "5pt" and cfg.cid == 1):
        return (math.cos(0.1 * t), math.sin(0.1 * t))
    if cfg.kind == "7pt":
        s = 1.0 + 0.1 * math.sin(t * cfg.dt)
        return (1.0 * s, 0.5 * s, 0.25 * s)
    return None


def initial_field(cfg: Config) -> np.ndarray:
    """u_0: sum of seeded Gaussian bumps (C1-C4); unused for C5 (b is fixed)."""
    if cfg.kind == "bsr":
        return np.zeros(cfg.n)
    nb, w, lo, hi = cfg.bumps
    u = np.empty(cfg.n)
    lib().sy_bumps(cfg.dim, cfg.N, nb, w, lo, hi, cfg.seed, _ptr(u))
    return u


def rhs(cfg: Config, u_prev: np.ndarray) -> np.ndarray:
    """b_t = u_{t-1}/dt + f (C1-C4); C5: fixed seeded N(0,1)-like vector."""
    b = np.empty(cfg.n)
    if cfg.kind == "bsr":
        lib().sy_normal_vec(cfg.n, cfg.seed, 0xB, _ptr(b))
    else:
        lib().sy_rhs(cfg.n, _ptr(np.ascontiguousarray(u_prev, dtype=np.float64)), cfg.dt, cfg.forcing, _ptr(b))
    return b


class HostMatrix:
    """CSR (or BSR) arrays of one system, numpy, int32 indices / float64 values."""

    def __init__(self, fmt, n, row_ptr, col_idx, val, block=1):
        self.fmt, self.n, self.row_ptr, self.col_idx, self.val, self.block = fmt, n, row_ptr, col_idx, val, block

    @property
    def nnz(self):
        return int(self.col_idx.shape[0])

    def to_scipy(self):
        import scipy.sparse as sp
        if self.fmt == "bsr":
            B = self.block
            data = self.val.reshape(-1, B, B).transpose(0, 2, 1)  # column-major blocks -> row-major
            return sp.bsr_matrix((data, self.col_idx, self.row_ptr), shape=(self.n, self.n)).tocsr()
        return sp.csr_matrix((self.val, self.col_idx, self.row_ptr), shape=(self.n, self.n))


class HostSequence:
    """Host generator of the sequence A_t, b_t (t = 1, 2, ...) of one config."""

    def __init__(self, cfg: Config):
        self.cfg = cfg
        L = lib()
        N = cfg.N
        n = cfg.n
        self.n = n
        if cfg.kind == "bsr":
            E = N
            nb = E ** 3
            nnzb = L.sy_c5_pattern(E, None, None, None)
            self.row_ptr = np.empty(nb + 1, np.int32)
            self.col_idx = np.empty(nnzb, np.int32)
            self.kind = np.empty(nnzb, np.int8)
            L.sy_c5_pattern(E, _ptr(self.row_ptr, _i32p), _ptr(self.col_idx, _i32p),
                            self.kind.ctypes.data_as(ctypes.POINTER(ctypes.c_int8)))
            self._base = None
            self._cur_t = 0
            self._cur = None
            return
        h = 1.0 / (N + 1)
        self.h = h
        nnz = nnz_closed_form(cfg)
        self.row_ptr = np.empty(n + 1, np.int32)
        self.col_idx = np.empty(nnz, np.int32)
        val = np.empty(nnz)
        self._fill(1, initial_field(cfg), self.row_ptr, self.col_idx, val)
        self._fixed = val if cfg.kind == "9pt" else None

    # scalars shared with the device generator (computed once, on the host)
    def scalars(self):
        cfg, h = self.cfg, self.h
        return dict(cd=cfg.nu / (h * h), ih=1.0 / h, idt=1.0 / cfg.dt, cdif=cfg.nu / (12.0 * h * h),
                    c6=1.0 / (6.0 * h))

    def _fill(self, t, u_prev, rp, ci, val):
        cfg, L, N = self.cfg, lib(), self.cfg.N
        sc = self.scalars()
        rpp = _ptr(rp, _i32p) if rp is not None else None
        cip = _ptr(ci, _i32p) if ci is not None else None
        if cfg.kind == "5pt":
            if cfg.cid == 2:
                uv = np.ascontiguousarray(u_prev, dtype=np.float64)
                L.sy_fill5(N, sc["cd"], sc["ih"], sc["idt"], 0.0, 0.0, _ptr(uv), rpp, cip, _ptr(val))
            else:
                bx, by = velocity(cfg, t)
                L.sy_fill5(N, sc["cd"], sc["ih"], sc["idt"], bx, by, None, rpp, cip, _ptr(val))
        elif cfg.kind == "9pt":
            L.sy_fill9(N, self.h, sc["cdif"], sc["c6"], sc["idt"], rpp, cip, _ptr(val))
        elif cfg.kind == "7pt":
            bx, by, bz = velocity(cfg, t)
            L.sy_fill7(N, sc["cd"], sc["ih"], sc["idt"], bx, by, bz, rpp, cip, _ptr(val))

    def matrix(self, t: int, u_prev: np.ndarray | None = None) -> HostMatrix:
        """A_t (t >= 1); u_prev = x_{t-1} is needed by C2 only."""
        cfg = self.cfg
        if cfg.kind == "bsr":
            return HostMatrix("bsr", self.n, self.row_ptr, self.col_idx, self._bsr_values(t), cfg.B)
        if self._fixed is not None:
            return HostMatrix("csr", self.n, self.row_ptr, self.col_idx, self._fixed)
        val = np.empty(self.col_idx.shape[0])
        self._fill(t, u_prev, None, None, val)
        return HostMatrix("csr", self.n, self.row_ptr, self.col_idx, val)

    def _bsr_values(self, t):
        cfg, L, B = self.cfg, lib(), self.cfg.B
        if self._base is None:
            nnzb = self.col_idx.shape[0]
            self._base = np.empty(nnzb * B * B)
            L.sy_c5_values(nnzb, B, cfg.seed, self.kind.ctypes.data_as(ctypes.POINTER(ctypes.c_int8)),
                           0.1 * 1.5, 0.1 * 0.5, _ptr(self._base))
        if self._cur is None or self._cur_t > t:
            self._cur = self._base.copy()
            self._cur_t = 1
        while self._cur_t < t:
            self._cur_t += 1
            L.sy_c5_perturb(self._cur.shape[0], cfg.seed, self._cur_t, _ptr(self._cur))
        return self._cur.copy()

    def rhs(self, t: int, u_prev: np.ndarray) -> np.ndarray:
        return rhs(self.cfg, u_prev)

    def initial(self) -> np.ndarray:
        return initial_field(self.cfg)


class DeviceSequence:
    """Device (torch/CUDA) generator of the same sequence, bit-identical to HostSequence.

    Pattern and fixed values are generated on the host once and copied; the per-system values
    and right-hand sides are produced by ``libsynth_cuda.so`` kernels from device-resident
    ``x_{t-1}``.
    """

    def __init__(self, cfg: Config, device="cuda", stream=None):
        import torch
        self.cfg = cfg
        self.torch = torch
        self.dev = device
        self.host = HostSequence(cfg)
        h = self.host
        self.row_ptr = torch.from_numpy(h.row_ptr).to(device)
        self.col_idx = torch.from_numpy(h.col_idx).to(device)
        self.n = cfg.n
        if cfg.kind == "bsr":
            self.kind = torch.from_numpy(h.kind).to(device)
            nnzb = h.col_idx.shape[0]
            self.val = torch.empty(nnzb * cfg.B * cfg.B, dtype=torch.float64, device=device)
            self._t = 0
        else:
            nnz = h.col_idx.shape[0]
            self.val = torch.empty(nnz, dtype=torch.float64, device=device)
            if cfg.kind == "9pt":
                self.val.copy_(torch.from_numpy(h._fixed))
        self.b = torch.empty(self.n, dtype=torch.float64, device=device)

    launches = 0  # device kernels launched by fill() (one per generator call)

    def _stream(self):
        return ctypes.c_void_p(self.torch.cuda.current_stream().cuda_stream)

    def fill(self, t: int, u_prev_dev, val_ptr=None):
        """Write A_t and b_t (into self.b) on the device, from device x_{t-1}.  The values go to
        self.val, or to the raw device pointer val_ptr (e.g. the solver's own buffer from
        rg_matrix_values, which then must hold A_{t-1} for the C5 multiplicative update)."""
        cfg, C, st = self.cfg, culib(), self._stream()
        vp = ctypes.c_void_p
        dst = vp(val_ptr if val_ptr is not None else self.val.data_ptr())
        if cfg.kind == "bsr":
            if self._t == 0 or t < self._t:
                self.launches += 1
                C.syd_c5_values(self.host.col_idx.shape[0], cfg.B, cfg.seed, vp(self.kind.data_ptr()),
                                0.1 * 1.5, 0.1 * 0.5, dst, st)
                self._t = 1
                self.launches += 1
                C.syd_normal_vec(self.n, cfg.seed, 0xB, vp(self.b.data_ptr()), st)
            while self._t < t:
                self._t += 1
                self.launches += 1
                C.syd_c5_perturb(self.val.numel(), cfg.seed, self._t, dst, st)
            return
        sc = self.host.scalars()
        if cfg.kind == "5pt":
            if cfg.cid == 2:
                self.launches += 1
                C.syd_fill5_values(cfg.N, sc["cd"], sc["ih"], sc["idt"], 0.0, 0.0, vp(u_prev_dev.data_ptr()),
                                   vp(self.row_ptr.data_ptr()), dst, st)
            else:
                bx, by = velocity(cfg, t)
                self.launches += 1
                C.syd_fill5_values(cfg.N, sc["cd"], sc["ih"], sc["idt"], bx, by, None,
                                   vp(self.row_ptr.data_ptr()), dst, st)
        elif cfg.kind == "7pt":
            bx, by, bz = velocity(cfg, t)
            self.launches += 1
            C.syd_fill7_values(cfg.N, sc["cd"], sc["ih"], sc["idt"], bx, by, bz,
                               vp(self.row_ptr.data_ptr()), dst, st)
        self.launches += 1
        C.syd_rhs(self.n, vp(u_prev_dev.data_ptr()), cfg.dt, cfg.forcing, vp(self.b.data_ptr()), st)
