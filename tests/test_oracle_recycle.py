"""Pins for the oracle's recycled variants (oracle.c or_solve augment/deflate, or_lsproj).

augment : min over x_c + span(W) + K_j(A, r_c)        (eqs def_aug_S/C_space)
deflate : min over x_c + span(W) + K_j(P A, P r_c)    (Table 1 row 6 "deflated LS", :348;
          P = I - AW((AW)^T AW)^{-1}(AW)^T, :310;  = GCRO inner iteration, :332)
"""
import numpy as np
import pytest

import oracle
from bruteforce import ls_projector, random_nonsym, restarted_minres


def _orthonormal(n, k, rng):
    Q, _ = np.linalg.qr(rng.standard_normal((n, k)))
    return Q


@pytest.mark.parametrize("variant", ["augment", "deflate"])
@pytest.mark.parametrize("m,k", [(5, 3), (9, 1), (4, 6)])
def test_matches_brute_force_explicit_space(rng, variant, m, k):
    """Residual at every step = explicit lstsq minimum over the stated space (restarts included)."""
    n = 36
    D = random_nonsym(n, rng, shift=1.4)
    W = _orthonormal(n, k, rng)
    b = rng.standard_normal(n)
    r = oracle.solve(oracle.Matrix.from_dense(D), b, m=m, variant=variant, W=W, tol=1e-9, max_iters=400)
    xb, itb, hb = restarted_minres(D, b, m, variant=variant, W=W, tol=1e-9, max_iters=400)
    assert r["iterations"] == itb
    kk = min(len(hb), len(r["history"]))
    assert np.allclose(r["history"][:kk], hb[:kk], rtol=1e-7, atol=1e-12)
    assert np.linalg.norm(r["x"] - xb) <= 1e-7 * np.linalg.norm(xb)
    assert r["converged"]


@pytest.mark.parametrize("variant", ["augment", "deflate"])
def test_rhs_in_image_of_recycle_space(rng, variant):
    """b = A W c  =>  the start projection already solves the system: x = W c, 0 iterations."""
    n, k = 30, 4
    D = random_nonsym(n, rng)
    W = _orthonormal(n, k, rng)
    c = rng.standard_normal(k)
    r = oracle.solve(oracle.Matrix.from_dense(D), D @ W @ c, m=10, variant=variant, W=W)
    assert r["iterations"] == 0 and r["converged"]
    assert np.linalg.norm(r["x"] - W @ c) <= 1e-12 * np.linalg.norm(c)


@pytest.mark.parametrize("variant", ["augment", "deflate"])
def test_empty_recycle_space_is_plain(rng, variant):
    n = 30
    D = random_nonsym(n, rng, shift=1.5)
    b = rng.standard_normal(n)
    A = oracle.Matrix.from_dense(D)
    p = oracle.solve(A, b, m=6, variant="plain")
    q = oracle.solve(A, b, m=6, variant=variant, W=None)
    assert p["iterations"] == q["iterations"]
    assert np.array_equal(p["x"], q["x"])


def test_projector_idempotent_and_annihilates_AW(rng):
    """P(Pw) = Pw and P A W = 0 (PAPER.md:239 'by construction M_D A V_s = 0' for the LS projector)."""
    n, k = 40, 5
    D = random_nonsym(n, rng)
    W = _orthonormal(n, k, rng)
    A = oracle.Matrix.from_dense(D)
    w = rng.standard_normal(n)
    Pw = oracle.lsproj(A, W, w)
    assert np.linalg.norm(oracle.lsproj(A, W, Pw) - Pw) <= 1e-14 * np.linalg.norm(w)
    PAW = oracle.lsproj(A, W, D @ W)
    assert np.linalg.norm(PAW) <= 1e-12 * np.linalg.norm(D) * np.linalg.norm(W)
    # equals the literal formula of Table 1 row 6
    assert np.allclose(Pw, ls_projector(D, W) @ w, rtol=0, atol=1e-12 * np.linalg.norm(w))


def test_deflated_residual_equals_true_residual(rng):
    """After the start projection P r_c = r_c, so the deflated min residual is the true one."""
    n, k = 36, 3
    D = random_nonsym(n, rng, shift=1.5)
    W = _orthonormal(n, k, rng)
    b = rng.standard_normal(n)
    r = oracle.solve(oracle.Matrix.from_dense(D), b, m=50, variant="deflate", W=W, tol=1e-10)
    assert abs(np.linalg.norm(b - D @ r["x"]) / np.linalg.norm(b) - r["history"][-1]) <= 1e-12


def test_invariant_subspace_estimate(rng):
    """Eq. estimate_deflation_vs_augmentation: for an A-invariant V_s the
    augmented residual has no V_s component (in exact arithmetic)."""
    n, k = 24, 3
    Q = _orthonormal(n, n, rng)
    T = np.triu(rng.standard_normal((n, n)) * 0.2) + np.diag(np.linspace(1.0, 3.0, n))
    D = Q @ T @ Q.T            # span(Q[:, :k]) is invariant under D (T upper triangular)
    W = Q[:, :k]
    b = rng.standard_normal(n)
    A = oracle.Matrix.from_dense(D)
    ra = oracle.solve(A, b, m=4, variant="augment", W=W, tol=1e-30, max_iters=4)
    res = b - D @ ra["x"]
    PV = W @ W.T
    assert np.linalg.norm(PV @ res) <= 1e-10 * np.linalg.norm(b)


def test_singular_recycle_space_raises(rng):
    n = 10
    D = random_nonsym(n, rng)
    w = rng.standard_normal(n)
    W = np.column_stack([w, 2 * w])
    with pytest.raises(np.linalg.LinAlgError):
        oracle.solve(oracle.Matrix.from_dense(D), rng.standard_normal(n), variant="deflate", W=W)
