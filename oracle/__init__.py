"""CPU oracle — TEST INFRASTRUCTURE ONLY.

Thin ctypes/numpy wrapper over ``oracle/liboracle.so`` (plain C99, fp64, deterministic OpenMP threads
over a fixed 256-chunk partition, so results do not depend on the thread count; see
``oracle.c`` for the definitions it follows and the PAPER.md passages it cites).  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference``
legs may import this package.  The product library (``paper_1807_09467_b200``) never does.

Parity status of each function:
  spmv / spmv_row     pinned: identity, diagonal, dense brute force (tests/test_oracle_spmv.py)
  solve (plain)       pinned: I, 2I, dense LU, restart = n termination, Arnoldi/monotonicity
  solve_basis         pinned: Arnoldi relation A V = V_{J+1} H (plain, augment) and the GCRO relation
                      A V = U_C B + V_{J+1} H (deflate) with A V formed by scipy.sparse; V^T V = I,
                      U_C^T V = 0 (tests/test_oracle_basis.py)
  threads             1 thread == N threads bitwise (solve, svd, spmv; tests/test_oracle_basis.py)
  solve (aug/defl)    pinned: brute-force dense least squares over the explicit space, b = A W c
                      special case, k = 0 reduces to plain, Table-1 row-6 projector properties
  solve (oblique)     pinned: brute-force dense least squares over the explicit monomial Krylov
                      space K_j(M_D A, M_D r_0), rows 2 = 5 (eq. equivalence_oblique), b = A W c
                      special case, W^T r = 0 on return, dense LU solution; obproj pinned by the
                      projector's defining properties (M_D A W = 0, W^T M_D = 0, M_D^2 = M_D, rank)
  solve (orthogonal)  pinned: brute-force lstsq over the explicit Krylov space of (I - WW^T) A
                      (rows 1 and 4, restarts, with the R19 per-cycle Galerkin completion), row 1 =
                      row 4, b = AWc, W^T r = 0 on return, LU solution
  ssor / solve(precond) pinned: M^{-1} equals the inverse of the explicitly assembled SSOR matrix
                      (D + wL) D^{-1} (D + wU)/(w(2-w)) of the permuted matrix, w = 1 diagonal A
                      closed form, symmetric A -> symmetric M^{-1}, triangular A in the order ->
                      forward sweep exact; right-preconditioned solves = lstsq over the explicit
                      space x_c + [span W] + M^{-1} K_j(op A M^{-1}, v) (all variants)
  svd / recycle_basis pinned: [3,4,0] closed form, orthonormal input, Eckart-Young tail,
                      numpy.linalg.svd brute force
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

_i32p = ctypes.POINTER(ctypes.c_int32)
_f64p = ctypes.POINTER(ctypes.c_double)

PLAIN, AUGMENT, DEFLATE, OBLIQUE, OBLIQUE_AUG, ORTHOGONAL, ORTHOGONAL_AUG = 0, 1, 2, 3, 4, 5, 6
# "oblique" = Table 1 row 5 (deflated oblique), "oblique_aug" = row 2 (augmented oblique),
# "orthogonal" = row 4 (deflated orthogonal), "orthogonal_aug" = row 1 (augmented orthogonal)
VARIANTS = {"plain": PLAIN, "augment": AUGMENT, "deflate": DEFLATE, "oblique": OBLIQUE,
            "oblique_aug": OBLIQUE_AUG, "orthogonal": ORTHOGONAL, "orthogonal_aug": ORTHOGONAL_AUG}


class _Mat(ctypes.Structure):
    _fields_ = [("fmt", ctypes.c_int), ("n", ctypes.c_int64), ("b", ctypes.c_int32),
                ("rp", _i32p), ("ci", _i32p), ("v", _f64p)]


class _Rep(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int), ("cycles", ctypes.c_int), ("converged", ctypes.c_int),
                ("status", ctypes.c_int), ("hist_len", ctypes.c_int), ("k_used", ctypes.c_int),
                ("rel_residual", ctypes.c_double)]


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run __graft_entry__.build() (or `make oracle`)")
        L = ctypes.CDLL(path)
        L.or_spmv.restype = None
        L.or_spmv.argtypes = [ctypes.POINTER(_Mat), _f64p, _f64p]
        L.or_spmv_row.restype = ctypes.c_double
        L.or_spmv_row.argtypes = [ctypes.POINTER(_Mat), ctypes.c_int64, _f64p]
        L.or_solve.restype = ctypes.c_int
        L.or_solve.argtypes = [ctypes.POINTER(_Mat), _f64p, _f64p, ctypes.c_int, ctypes.c_int, _f64p,
                               ctypes.c_int, ctypes.c_double, ctypes.c_int, _f64p, ctypes.POINTER(_Rep),
                               _f64p, ctypes.c_int]
        L.or_solve_pc.restype = ctypes.c_int
        L.or_solve_pc.argtypes = L.or_solve.argtypes + [_i32p, ctypes.c_double]
        L.or_ssor.restype = ctypes.c_int
        L.or_ssor.argtypes = [ctypes.POINTER(_Mat), _i32p, ctypes.c_double, _f64p, _f64p]
        L.or_lsproj.restype = ctypes.c_int
        L.or_lsproj.argtypes = [ctypes.POINTER(_Mat), _f64p, ctypes.c_int, _f64p, ctypes.c_int]
        L.or_obproj.restype = ctypes.c_int
        L.or_obproj.argtypes = [ctypes.POINTER(_Mat), _f64p, ctypes.c_int, _f64p, ctypes.c_int]
        L.or_solve_basis.restype = ctypes.c_int
        L.or_solve_basis.argtypes = [ctypes.POINTER(_Mat), _f64p, _f64p, ctypes.c_int, ctypes.c_int, _f64p,
                                     ctypes.c_int, ctypes.c_double, ctypes.c_int, _f64p, ctypes.POINTER(_Rep),
                                     _f64p, _f64p, _f64p, ctypes.POINTER(ctypes.c_int)]
        L.or_set_threads.restype = None
        L.or_set_threads.argtypes = [ctypes.c_int]
        L.or_get_threads.restype = ctypes.c_int
        L.or_get_threads.argtypes = []
        L.or_svd.restype = ctypes.c_int
        L.or_svd.argtypes = [ctypes.c_int64, ctypes.c_int, _f64p, ctypes.c_int64, _f64p, _f64p,
                             ctypes.POINTER(ctypes.c_int)]
        _LIB = L
    return _LIB


def _f(a):
    return a.ctypes.data_as(_f64p)


def set_threads(t: int):
    """Threads the oracle may use (results do not depend on it: fixed 256-chunk partition)."""
    lib().or_set_threads(int(t))


def threads() -> int:
    return int(lib().or_get_threads())


class Matrix:
    """A CSR (fmt='csr') or BSR (fmt='bsr', column-major b x b blocks) matrix held by numpy arrays."""

    def __init__(self, n, row_ptr, col_idx, val, fmt="csr", block=1):
        self.n = int(n)
        self.fmt = fmt
        self.block = int(block)
        self.row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int32)
        self.col_idx = np.ascontiguousarray(col_idx, dtype=np.int32)
        self.val = np.ascontiguousarray(val, dtype=np.float64)
        self._m = _Mat(0 if fmt == "csr" else 1, self.n, self.block,
                       self.row_ptr.ctypes.data_as(_i32p), self.col_idx.ctypes.data_as(_i32p), _f(self.val))

    @classmethod
    def from_host(cls, hm):
        """From a synth.HostMatrix."""
        return cls(hm.n, hm.row_ptr, hm.col_idx, hm.val, hm.fmt, hm.block)

    @classmethod
    def from_dense(cls, D):
        D = np.asarray(D, dtype=np.float64)
        n = D.shape[0]
        rp, ci, v = [0], [], []
        for i in range(n):
            for j in range(n):
                if D[i, j] != 0.0:
                    ci.append(j)
                    v.append(D[i, j])
            rp.append(len(ci))
        return cls(n, np.array(rp), np.array(ci, dtype=np.int32), np.array(v))


def spmv(A: Matrix, x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty(A.n)
    lib().or_spmv(ctypes.byref(A._m), _f(x), _f(y))
    return y


def spmv_row(A: Matrix, row: int, x: np.ndarray) -> float:
    x = np.ascontiguousarray(x, dtype=np.float64)
    return lib().or_spmv_row(ctypes.byref(A._m), int(row), _f(x))


def ssor_order(colors):
    """Row order of a multicolour SSOR: rows sorted by colour, natural order inside a colour."""
    colors = np.asarray(colors)
    return np.ascontiguousarray(np.argsort(colors, kind="stable"), dtype=np.int32)


def ssor(A: Matrix, order, omega, z):
    """M^{-1} z for SSOR(omega) in the given row order (oracle.c or_ssor)."""
    order = np.ascontiguousarray(order, dtype=np.int32)
    z = np.ascontiguousarray(z, dtype=np.float64)
    out = np.empty(A.n)
    if lib().or_ssor(ctypes.byref(A._m), order.ctypes.data_as(_i32p), float(omega), _f(z), _f(out)):
        raise np.linalg.LinAlgError("oracle: zero diagonal entry")
    return out


def solve(A: Matrix, b, x0=None, m=30, variant="plain", W=None, tol=1e-8, max_iters=20000,
          hist_cap=None, precond=None):
    """Restarted min-residual solve (plain / augment / deflate / oblique / oblique_aug).  W: n x k
    array (columns span the recycle space) or None.  precond: None or (order, omega) = right SSOR
    preconditioner in that row order.  Returns dict(x, iterations, cycles, converged, rel_residual,
    history)."""
    v = VARIANTS[variant] if isinstance(variant, str) else int(variant)
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.empty(A.n)
    k = 0
    Wf = None
    if W is not None and v != PLAIN:
        W = np.asarray(W, dtype=np.float64)
        if W.ndim == 1:
            W = W[:, None]
        k = W.shape[1]
        Wf = np.asfortranarray(W)
    hist_cap = hist_cap or max_iters
    hist = np.empty(hist_cap)
    rep = _Rep()
    x0p = None
    if x0 is not None:
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        x0p = _f(x0)
    args = [ctypes.byref(A._m), _f(b), x0p, int(m), v, Wf.ctypes.data_as(_f64p) if Wf is not None and k > 0 else None,
            k, float(tol), int(max_iters), _f(x), ctypes.byref(rep), _f(hist), hist_cap]
    if precond is None:
        st = lib().or_solve(*args)
    else:
        order = np.ascontiguousarray(precond[0], dtype=np.int32)
        st = lib().or_solve_pc(*args, order.ctypes.data_as(_i32p), float(precond[1]))
    if st == 1:
        raise np.linalg.LinAlgError("oracle: A W is (numerically) rank deficient" if v < OBLIQUE
                                    else "oracle: E = W^T A W is (numerically) singular")
    if st == 3:
        raise np.linalg.LinAlgError("oracle: zero diagonal entry (SSOR)")
    if st != 0:
        raise MemoryError("oracle: allocation failed")
    return dict(x=x, iterations=rep.iterations, cycles=rep.cycles, converged=bool(rep.converged),
                rel_residual=rep.rel_residual, history=hist[:rep.hist_len].copy(), k_used=rep.k_used)


def solve_basis(A: Matrix, b, x0=None, m=30, variant="plain", W=None, tol=1e-8, max_iters=20000):
    """As solve (plain / augment / deflate, no preconditioner), also returning the LAST restart
    cycle's Krylov basis: V (n x J, orthonormal v_0..v_{J-1}), H (J+1 x J upper Hessenberg: the
    Arnoldi coefficients) and, for deflate, B (k x J: U_C^T A v_j against the orthonormal basis of
    A W), so that A V = V_{J+1} H (plain, augment) / A V = U_C B + V_{J+1} H (deflate), where
    v_J is the un-returned next vector (its coefficient is H[J, J-1])."""
    v = VARIANTS[variant] if isinstance(variant, str) else int(variant)
    if v not in (PLAIN, AUGMENT, DEFLATE):
        raise ValueError("solve_basis: plain, augment or deflate")
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.empty(A.n)
    k, Wf = 0, None
    if W is not None and v != PLAIN:
        W = np.asarray(W, dtype=np.float64).reshape(A.n, -1)
        k = W.shape[1]
        Wf = np.asfortranarray(W)
    V = np.zeros((A.n, m), order="F")
    H = np.zeros((m + 1, m), order="F")
    B = np.zeros((max(k, 1), m), order="F")
    rep = _Rep()
    steps = ctypes.c_int(0)
    x0p = None
    if x0 is not None:
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        x0p = _f(x0)
    st = lib().or_solve_basis(ctypes.byref(A._m), _f(b), x0p, int(m), v,
                              Wf.ctypes.data_as(_f64p) if k > 0 else None, k, float(tol), int(max_iters), _f(x),
                              ctypes.byref(rep), V.ctypes.data_as(_f64p), H.ctypes.data_as(_f64p),
                              B.ctypes.data_as(_f64p), ctypes.byref(steps))
    if st == 1:
        raise np.linalg.LinAlgError("oracle: A W is (numerically) rank deficient")
    if st != 0:
        raise MemoryError("oracle: allocation failed")
    J = steps.value
    return dict(x=x, iterations=rep.iterations, cycles=rep.cycles, converged=bool(rep.converged),
                rel_residual=rep.rel_residual, steps=J, V=np.ascontiguousarray(V[:, :J]),
                H=np.ascontiguousarray(H[:J + 1, :J]), B=np.ascontiguousarray(B[:k, :J]))


def lsproj(A: Matrix, W, Z):
    """P Z with P = I - AW((AW)^T AW)^{-1}(AW)^T, computed as the oracle's solver
    does (MGS2 QR of AW).  Z: n-vector or n x q array."""
    W = np.asfortranarray(np.asarray(W, dtype=np.float64).reshape(A.n, -1))
    Z = np.asarray(Z, dtype=np.float64)
    one = Z.ndim == 1
    Zf = np.asfortranarray(Z.reshape(A.n, -1)).copy(order="F")
    st = lib().or_lsproj(ctypes.byref(A._m), W.ctypes.data_as(_f64p), W.shape[1], Zf.ctypes.data_as(_f64p),
                         Zf.shape[1])
    if st:
        raise np.linalg.LinAlgError("oracle: A W is (numerically) rank deficient")
    return Zf[:, 0].copy() if one else Zf


def obproj(A: Matrix, W, Z):
    """M_D Z with M_D = I - A W E^{-1} W^T, E = W^T A W (eq. left_deflation),
    computed as the oracle's oblique solver does (LU of E).  Z: n-vector or n x q array."""
    W = np.asfortranarray(np.asarray(W, dtype=np.float64).reshape(A.n, -1))
    Z = np.asarray(Z, dtype=np.float64)
    one = Z.ndim == 1
    Zf = np.asfortranarray(Z.reshape(A.n, -1)).copy(order="F")
    st = lib().or_obproj(ctypes.byref(A._m), W.ctypes.data_as(_f64p), W.shape[1], Zf.ctypes.data_as(_f64p),
                         Zf.shape[1])
    if st:
        raise np.linalg.LinAlgError("oracle: E = W^T A W is (numerically) singular")
    return Zf[:, 0].copy() if one else Zf


def svd(X):
    """Thin SVD of X (n x s) by one-sided Jacobi: returns (U, sigma, rank, sweeps)."""
    X = np.asfortranarray(np.asarray(X, dtype=np.float64))
    if X.ndim == 1:
        X = X[:, None]
    n, s = X.shape
    U = np.empty((n, s), order="F")
    sig = np.empty(s)
    rk = ctypes.c_int(0)
    sweeps = lib().or_svd(n, s, X.ctypes.data_as(_f64p), n, U.ctypes.data_as(_f64p), _f(sig), ctypes.byref(rk))
    return U, sig, rk.value, sweeps


def recycle_basis(X, k, modes="largest"):
    """Algorithm 1: V_s = first k left singular vectors of the window X
    ("largest"), or the k smallest NON-ZERO ones ("smallest", the alternative of PAPER.md:673-676:
    "the SVD modes with smaller singular values"), with k_eff = min(k, #columns, rank) where
    rank = #{sigma > 1e-12 sigma_1}.  Returns (W, sigma, k_eff)."""
    U, sig, rank, _ = svd(X)
    k_eff = min(int(k), U.shape[1], rank)
    if modes == "smallest":
        return np.ascontiguousarray(U[:, rank - k_eff:rank]), sig, k_eff
    return np.ascontiguousarray(U[:, :k_eff]), sig, k_eff
