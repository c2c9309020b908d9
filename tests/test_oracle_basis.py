"""Pins for the oracle's Krylov basis and its deterministic threading.

The basis invariants named by BASELINE.json's north star and SURVEY.md §8(c) (lines "A V_m =
V_{m+1} H_m", "V orthonormal to 1e-12", GCRO relation "A V_m = Q B_m + V_{m+1} H_m", "Q^T V = 0"):
an orthogonal Krylov basis, the non-naive iterate computation that relies on the
Arnoldi relation, and the GCRO equivalence of deflation.  A V is
formed here by scipy.sparse (not by the oracle's SpMV) and V_{J+1} H by numpy, so a dropped term,
a wrong index or a transposed operand in the oracle's Arnoldi fails one of these.

Threading: the oracle's fixed 256-chunk partition makes every result bitwise
independent of the thread count.
"""
import numpy as np
import pytest
import scipy.sparse as sp

import oracle
import synth
from bruteforce import random_nonsym


def _csr(D):
    return oracle.Matrix.from_dense(D)


def _next_vector(A_s, V, H, B=None, U=None):
    """v_J implied by the last column: (A v_{J-1} - U b - V h) / H[J, J-1] (from the relation)."""
    J = V.shape[1]
    w = A_s @ V[:, J - 1] - V @ H[:J, J - 1]
    if B is not None and B.size:
        w -= U @ B[:, J - 1]
    return w / H[J, J - 1]


def _check_relation(A_s, V, H, B=None, U=None, tol=1e-12):
    J = V.shape[1]
    assert J >= 2
    # orthonormality of v_0..v_{J-1}, and of the implied v_J
    vJ = _next_vector(A_s, V, H, B, U)
    V1 = np.column_stack([V, vJ])
    assert np.max(np.abs(V1.T @ V1 - np.eye(J + 1))) <= tol
    # the relation over the first J-1 columns (uses only returned columns)
    AV = A_s @ V[:, : J - 1]
    rhs = V @ H[:J, : J - 1]
    if B is not None and B.size:
        rhs = rhs + U @ B[:, : J - 1]
    A_F = sp.linalg.norm(A_s)
    assert np.linalg.norm(AV - rhs) <= tol * A_F * np.sqrt(J)
    # H upper Hessenberg with a positive sub-diagonal
    assert np.all(np.tril(H, -2) == 0.0)
    assert np.all(np.diag(H, -1) > 0.0)
    if U is not None and U.size:
        assert np.max(np.abs(U.T @ V1)) <= tol


@pytest.mark.parametrize("variant", ["plain", "augment"])
def test_arnoldi_relation_random(rng, variant):
    n, m = 60, 12
    D = random_nonsym(n, rng, shift=1.3)
    b = rng.standard_normal(n)
    W = np.linalg.qr(rng.standard_normal((n, 3)))[0] if variant == "augment" else None
    r = oracle.solve_basis(_csr(D), b, m=m, variant=variant, W=W, tol=1e-10)
    assert r["converged"]
    _check_relation(sp.csr_matrix(D), r["V"], r["H"])


def test_gcro_relation_deflate_random(rng):
    n, m, k = 60, 12, 4
    D = random_nonsym(n, rng, shift=1.3)
    b = rng.standard_normal(n)
    W = np.linalg.qr(rng.standard_normal((n, k)))[0]
    r = oracle.solve_basis(_csr(D), b, m=m, variant="deflate", W=W, tol=1e-10)
    assert r["converged"] and r["B"].shape == (k, r["steps"])
    U = np.linalg.qr(D @ W)[0]  # orthonormal basis of A W (numpy QR: independent of the oracle)
    # the oracle's U_C may differ from numpy's Q by column signs: B is checked through U B = U_C B
    sgn = np.sign(np.diag(np.linalg.qr(D @ W)[1]))
    _check_relation(sp.csr_matrix(D), r["V"], r["H"], r["B"], U * sgn)


@pytest.mark.parametrize("variant", ["plain", "deflate"])
def test_relation_on_c1_stencil(variant):
    """The same invariants on the C1 upwind convection-diffusion operator (BASELINE configs[0])."""
    cfg = synth.CONFIGS["C1"]
    seq = synth.HostSequence(cfg)
    u0 = seq.initial()
    M = seq.matrix(1, u0)
    A = oracle.Matrix.from_host(M)
    b = seq.rhs(1, u0)
    W = None
    if variant == "deflate":
        X = np.column_stack([np.sin((i + 1) * np.linspace(0, 3, cfg.n)) for i in range(cfg.k)])
        W = oracle.recycle_basis(X, cfg.k)[0]
    r = oracle.solve_basis(A, b, m=cfg.m, variant=variant, W=W, tol=cfg.tol)
    assert r["converged"]
    A_s = M.to_scipy()
    U = None
    if variant == "deflate":
        Q, R = np.linalg.qr(A_s @ W)
        U = Q * np.sign(np.diag(R))
    _check_relation(A_s, r["V"], r["H"], r["B"] if variant == "deflate" else None, U)


def test_basis_is_last_cycle_and_matches_solve(rng):
    """solve_basis gives the same x / iterations as solve (the export does not perturb the solve)."""
    n = 80
    D = random_nonsym(n, rng, shift=1.1)
    b = rng.standard_normal(n)
    A = _csr(D)
    r1 = oracle.solve(A, b, m=6, tol=1e-9)
    r2 = oracle.solve_basis(A, b, m=6, tol=1e-9)
    assert r1["iterations"] == r2["iterations"] and r2["cycles"] > 1
    assert np.array_equal(r1["x"], r2["x"])
    assert r2["steps"] == r1["iterations"] - 6 * (r1["cycles"] - 1)


def _big_system(n, rng):
    """A banded random non-symmetric system long enough for the threaded paths (n >= 65536)."""
    offs = [-257, -1, 0, 1, 256]
    diags = [rng.uniform(-1, 0, n - abs(o)) for o in offs]
    diags[2] = 5.0 + rng.random(n)
    A_s = sp.diags(diags, offs, format="csr")
    A_s.sort_indices()
    return oracle.Matrix(n, A_s.indptr, A_s.indices, A_s.data), A_s


def test_threads_bitwise_identical(rng):
    """1 thread and N threads: bitwise identical SpMV, solve (all three variants) and SVD."""
    n = 70000
    A, _ = _big_system(n, rng)
    b = rng.standard_normal(n)
    X = rng.standard_normal((n, 5))
    W = oracle.recycle_basis(X, 3)[0]
    nt0 = oracle.threads()
    out = {}
    try:
        for t in (1, 4):
            oracle.set_threads(t)
            y = oracle.spmv(A, b)
            rs = [oracle.solve(A, b, m=8, variant=v, W=W, tol=1e-10) for v in ("plain", "augment", "deflate")]
            U, sig, _, _ = oracle.svd(X)
            out[t] = (y, [(r["x"], r["iterations"], r["history"]) for r in rs], U, sig)
    finally:
        oracle.set_threads(nt0)
    a, c = out[1], out[4]
    assert np.array_equal(a[0], c[0])
    for (x1, i1, h1), (x2, i2, h2) in zip(a[1], c[1]):
        assert i1 == i2 and np.array_equal(x1, x2) and np.array_equal(h1, h2)
    assert np.array_equal(a[2], c[2]) and np.array_equal(a[3], c[3])


def test_threaded_relation_large(rng):
    """The basis invariants also hold on the threaded path (n above the parallel threshold)."""
    n = 70000
    A, A_s = _big_system(n, rng)
    b = rng.standard_normal(n)
    r = oracle.solve_basis(A, b, m=10, tol=1e-10)
    _check_relation(A_s, r["V"], r["H"])
